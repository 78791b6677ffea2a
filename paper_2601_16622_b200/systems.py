"""Synthetic atom systems of the benchmark configurations (host side).

gen_fcc_system follows SPEC.md:422-430,466: sample N
sites without replacement from the smallest cubic FCC supercell (4-site
basis, lattice constant a) holding >= N sites; open boundaries.  Sampled
sites are kept in lattice order (spatially coherent, good for the gather
locality of the attention kernels).  The SPEC's libstdc++ mt19937_64 stream
(rng.hpp:12) is not reproducible outside libstdc++; numpy's PCG64 seeded by
EQUISTREAM_SEED (else 0, rng.hpp:14-22) is used instead -- inputs are shared
byte-for-byte between the GPU path and the oracle, which is what parity needs.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

FCC_BASIS = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])


def default_seed(fallback: int = 0) -> int:
    try:
        return int(os.environ.get("EQUISTREAM_SEED", fallback))
    except ValueError:
        return fallback


def fcc_cells_for(n_atoms: int) -> int:
    n = 1
    while 4 * n ** 3 < n_atoms:
        n += 1
    return n


def fcc_sites(n: int, a: float) -> np.ndarray:
    g = np.arange(n, dtype=np.float64)
    cell = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 1, 3)
    return ((cell + FCC_BASIS[None]) * a).reshape(-1, 3)


def gen_fcc_system(n_atoms: int, a: float = 3.8, seed: int = 0, n_cells: int | None = None) -> np.ndarray:
    """Positions [N, 3] float64."""
    if n_atoms < 1:
        raise ValueError("gen_fcc_system: N >= 1")
    n = fcc_cells_for(n_atoms) if n_cells is None else n_cells
    sites = fcc_sites(n, a)
    if n_atoms > len(sites):
        raise ValueError("gen_fcc_system: supercell too small")
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(len(sites), size=n_atoms, replace=False))
    return np.ascontiguousarray(sites[pick])


@dataclass
class System:
    pos: np.ndarray                      # [N, 3] float64
    seg_ptr: np.ndarray | None = None    # [B+1] int32 molecule offsets, None = one system
    box: np.ndarray | None = None        # [3] periodic box (minimum image), None = open
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_atoms(self) -> int:
        return int(self.pos.shape[0])


def molecule_batch(n_mol: int, lo: int, hi: int, seed: int = 0, a: float = 3.8, seed_offset: int = 1000,
                   fixed: int | None = None) -> System:
    """Config 2/4: a batch of independent molecules; no cross-molecule pairs."""
    rng = np.random.default_rng(seed)
    sizes = np.full(n_mol, fixed) if fixed is not None else rng.integers(lo, hi + 1, size=n_mol)
    parts = [gen_fcc_system(int(s), a, seed + seed_offset + m) for m, s in enumerate(sizes)]
    seg = np.zeros(n_mol + 1, dtype=np.int32)
    seg[1:] = np.cumsum(sizes)
    return System(np.ascontiguousarray(np.concatenate(parts)), seg, None, f"batch{n_mol}",
                  {"sizes": sizes})


def periodic_box(n_atoms: int, n_cells: int = 30, a: float = 3.8, seed: int = 0) -> System:
    """Config 5: N of the 4 n^3 sites of an n-cell FCC box under PBC."""
    pos = gen_fcc_system(n_atoms, a, seed, n_cells=n_cells)
    return System(pos, None, np.full(3, n_cells * a), f"pbc{n_atoms}")


def config_system(cfg: int, seed: int = 0, n_atoms: int | None = None, n_mol: int | None = None) -> System:
    """The five BASELINE.json configurations (SURVEY.md §8 d)."""
    if cfg == 1:
        return System(gen_fcc_system(64, 3.8, seed), None, None, "mol64")
    if cfg == 2:
        return molecule_batch(n_mol or 4096, 40, 60, seed, seed_offset=1000)
    if cfg == 3:
        return System(gen_fcc_system(n_atoms or 20000, 3.8, seed), None, None, f"fcc{n_atoms or 20000}")
    if cfg == 4:
        return molecule_batch(n_mol or 256, 350, 350, seed, seed_offset=2000, fixed=350)
    if cfg == 5:
        return periodic_box(n_atoms or 100000, 30, 3.8, seed)
    raise ValueError(f"unknown config {cfg}")


CONFIG_SHAPES = {  # (L, C, H)
    1: (2, 64, 8),
    2: (2, 128, 8),
    3: (2, 128, 8),
    4: (4, 128, 8),
    5: (2, 128, 8),
}


def random_features(n_atoms: int, L: int, C: int, seed: int) -> np.ndarray:
    """h ~ N(0,1), [N][M][C] float64."""
    rng = np.random.default_rng(seed + 7)
    return rng.standard_normal((n_atoms, (L + 1) ** 2, C))


def random_weights(L: int, C: int, seed: int, dq: int | None = None, cv: int | None = None) -> np.ndarray:
    """Per-degree projection W [L+1][C][2Dq+Cv] ~ N(0, 1/C) (SURVEY §8 decisions)."""
    dq = 2 * C if dq is None else dq
    cv = C if cv is None else cv
    rng = np.random.default_rng(seed + 11)
    return rng.standard_normal((L + 1, C, 2 * dq + cv)) / np.sqrt(C)
