"""Condense an `ncu --set full` report into the per-kernel numbers the
roofline cites: duration, DRAM bytes (read + write) and throughput, SM /
tensor-pipe / issue utilisation, occupancy and the top stall reasons.

    python profiles/tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_summary.txt
    python profiles/tools/ncu_summary.py gpurun_out/prof.ncu-rep --json   (machine-readable)
    python profiles/tools/ncu_summary.py gpurun_out/prof.ncu-rep --traffic > profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor_pipe_pct"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_mem_pct"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "tmem_inst_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "registers"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        yield hdr, units, v


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main(rep, as_json, traffic=False):
    res = []
    for hdr, units, v in rows(rep):
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "?")[:90]}
        for k, name in KEYS:
            if k in d:
                e[name] = num(d[k])
                e[name + "_unit"] = u.get(k, "")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(d[k]) or 0.0) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(x for _, x in st) or 1.0
        e["stalls"] = {k: round(100 * x / tot, 1) for k, x in sorted(st, key=lambda t: -t[1])[:6]}
        res.append(e)
    if as_json:
        print(json.dumps(res, indent=1))
        return
    if traffic:  # profiles/ncu_traffic.json: what bench.py's roofline line reads (first launch of each kernel)
        out = {"source": f"{rep} (ncu --set full)", "bytes_per_launch": {}}
        for e in res:
            full = e["kernel"].split("(")[0].split("::")[-1].strip()
            name = full.split("<")[0]
            if name == "attn_dqk_tc_kernel":  # the two instances: <0> dq (query tiles), <1> dk (key tiles)
                name = "attn_dk_tc_kernel" if full.endswith("<1>") else "attn_dq_tc_kernel"
            if name in out["bytes_per_launch"]:
                continue
            byt = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            tns = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}
            rd = (e.get("dram_read") or 0) * byt.get(e.get("dram_read_unit", "byte"), 1)
            wr = (e.get("dram_write") or 0) * byt.get(e.get("dram_write_unit", "byte"), 1)
            out["bytes_per_launch"][name] = {
                "dram_read": round(rd), "dram_write": round(wr), "total": round(rd + wr),
                "tensor_pipe_pct": e.get("tensor_pipe_pct"),
                "duration_ns": round((e.get("duration") or 0) * tns.get(e.get("duration_unit", "nsecond"), 1))}
        print(json.dumps(out, indent=1))
        return
    for e in res:
        print(e["kernel"])
        for _, name in KEYS:
            if name in e and e[name] is not None:
                print(f"  {name:16s} {e[name]:>16,.2f} {e.get(name + '_unit', '')}")
        print("  stalls          ", ", ".join(f"{k} {x}%" for k, x in e["stalls"].items()))


if __name__ == "__main__":
    main(sys.argv[1], "--json" in sys.argv, "--traffic" in sys.argv)
