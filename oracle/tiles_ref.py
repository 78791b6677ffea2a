"""NumPy restatement of the tensor-core tile structures (es_attn_tiles_build,
north-star subsystem 3: "cell-list / radius-cutoff neighbour-tile builder and
tile-skip mask") -- TEST INFRASTRUCTURE ONLY, the checker of the GPU builder.

It states the structures from their definitions, not from the kernels:

* query tiles: 128 consecutive rows, or (molecule batches) whole segments
  packed greedily into tiles of at most 128 rows, segments longer than a tile
  split at 128-row boundaries; the greedy scan runs over `parts` consecutive
  groups of segments, each group starting a fresh tile;
* tile-skip mask: bit kb of tile t set iff a row of t lists a key in 16-key
  chunk kb; the tile's chunk list = its set bits, ascending; cptr = the
  exclusive prefix sum of the list lengths;
* per-row lists: one entry per distinct chunk the row touches, (position of
  the chunk in its tile's list) << 16 | (16-bit mask of the keys), ascending,
  then 0xffff0000 if the row has fewer than K entries;
* slots: the row's valid neighbour slots ordered by key index j (the order the
  per-row lists enumerate keys); rank_of[slot] = the slot's position there;
* key side (the dk pass): the same over the transposed relation -- tiles of
  key atoms, 16-query chunks, per-key entries stored at rev_ptr[j].
"""
from __future__ import annotations

import numpy as np

TQ, KC = 128, 16


def pack_parts(N: int) -> int:
    return min(1024, ((N + TQ - 1) // TQ) // 32 + 1)


def tile_starts(N: int, seg=None) -> list[int]:
    """First row of every non-empty tile (then N)."""
    if seg is None or len(seg) < 2:
        return list(range(0, N, TQ)) + [N]
    seg = [int(x) for x in seg]
    nseg = len(seg) - 1
    parts = pack_parts(N)
    G = (nseg + parts - 1) // parts
    starts = []
    for p in range(parts):
        s0, s1 = min(nseg, p * G), min(nseg, p * G + G)
        if s0 >= s1:
            continue
        cur = 0 if s0 == 0 else min(N, max(0, seg[s0]))
        starts.append(cur)
        lo = cur
        for x in range(s0, s1):
            hi = min(N, max(lo, seg[x + 1]))
            if hi - cur > TQ and lo > cur:
                cur = lo
                starts.append(cur)
            while hi - cur > TQ:
                cur += TQ
                starts.append(cur)
            lo = hi
    return starts + [N]


def build(nbr: np.ndarray, seg=None, n_keys: int | None = None):
    """Query-side structures of a neighbour table [N][K] (keys in [0, n_keys))."""
    N, K = nbr.shape
    Nk = N if n_keys is None else n_keys
    ts = tile_starts(N, seg)
    ntiles = len(ts) - 1
    rtile = np.zeros(N, np.int64)
    for t in range(ntiles):
        rtile[ts[t]:ts[t + 1]] = t
    chunks = [set() for _ in range(ntiles)]
    for i in range(N):
        for j in nbr[i]:
            if j >= 0:
                chunks[rtile[i]].add(int(j) // KC)
    clist = [sorted(c) for c in chunks]
    cptr = np.concatenate([[0], np.cumsum([len(c) for c in clist])]).astype(np.int64)
    rowlist = np.zeros((N, K), np.uint32)
    slots = np.full((N, K), -1, np.int64)
    rank_of = np.full((N, K), -1, np.int64)
    for i in range(N):
        pos = {c: u for u, c in enumerate(clist[rtile[i]])}
        valid = [(int(j), s) for s, j in enumerate(nbr[i]) if j >= 0]
        valid.sort()
        ents = {}
        for r, (j, s) in enumerate(valid):
            slots[i, r] = s
            rank_of[i, s] = r
            c = pos[j // KC]
            ents[c] = ents.get(c, 0) | (1 << (j % KC))
        ent = [(c << 16) | m for c, m in sorted(ents.items())]
        rowlist[i, :len(ent)] = ent
        if len(ent) < K:
            rowlist[i, len(ent)] = 0xFFFF0000
    return {"tstart": np.array(ts, np.int64), "rtile": rtile, "clist": clist, "cptr": cptr, "rowlist": rowlist,
            "slots": slots, "rank_of": rank_of, "nkb": (Nk + KC - 1) // KC}


def build_keys(nbr: np.ndarray, rev_ptr: np.ndarray, rev_pair: np.ndarray, seg=None, n_keys: int | None = None):
    """Key-side structures (tiles of key atoms, 16-query chunks)."""
    N, K = nbr.shape
    Nk = N if n_keys is None else n_keys
    ts = tile_starts(Nk, seg if Nk == N else None)
    ntiles = len(ts) - 1
    rtile = np.zeros(Nk, np.int64)
    for t in range(ntiles):
        rtile[ts[t]:ts[t + 1]] = t
    chunks = [set() for _ in range(ntiles)]
    for i in range(N):
        for j in nbr[i]:
            if j >= 0:
                chunks[rtile[j]].add(i // KC)
    clist = [sorted(c) for c in chunks]
    cptr = np.concatenate([[0], np.cumsum([len(c) for c in clist])]).astype(np.int64)
    rowlist = {}
    for j in range(Nk):
        e0, e1 = int(rev_ptr[j]), int(rev_ptr[j + 1])
        pos = {c: u for u, c in enumerate(clist[rtile[j]])}
        ents = {}
        for e in range(e0, e1):
            i = int(rev_pair[e]) // K
            c = pos[i // KC]
            ents[c] = ents.get(c, 0) | (1 << (i % KC))
        ent = [(c << 16) | m for c, m in sorted(ents.items())]
        if len(ent) < e1 - e0:
            ent.append(0xFFFF0000)
        rowlist[j] = np.array(ent, np.uint32)
    return {"tstart": np.array(ts, np.int64), "rtile": rtile, "clist": clist, "cptr": cptr, "rowlist": rowlist}
