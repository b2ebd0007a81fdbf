"""Summarise ncu outputs into markdown for profiles/.

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel device time (cold, serialised)
    python tools/ncu_summary.py full <report.ncu-rep>        # --set full key metrics per kernel
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% |")


KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("dram__bytes_read.sum", "DRAM read (B)"),
    ("dram__bytes_write.sum", "DRAM write (B)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    units = rows[1]
    print("| kernel | " + " | ".join(f"{k[1]} [{units[idx[k[0]]]}]" if k[0] in idx else k[1]
                                    for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        vals = [r[idx[k]] if k in idx else "" for k, _ in KEYS]
        print(f"| `{name}` | " + " | ".join(vals) + " |")


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
FAMILY = {"k_render_fwd": "render_fwd", "k_render_bwd": "render_bwd", "k_preprocess": "preprocess",
          "k_view_accumulate": "view_accumulate", "k_tomo_fwd": "tomo_fwd", "k_tomo_bwd": "tomo_bwd"}


def traffic(path, source="", config=None, out_path=None, view="0"):
    """Per-launch averages of the blend / preprocess kernels; with config and
    out_path, merged into that JSON under the config's key."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}

    def val(r, key):
        v = float(r[idx[key]].replace(",", ""))
        return v * SCALE.get(units[idx[key]], 1.0)
    acc = defaultdict(list)
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        if name in FAMILY:
            acc[FAMILY[name]].append(r)
    res = {}
    for fam, rs in acc.items():
        def mean(key, rs=rs):
            return sum(val(r, key) for r in rs) / len(rs)
        rd, wr = mean("dram__bytes_read.sum"), mean("dram__bytes_write.sum")
        res[fam] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                    "warp_instructions_per_launch": mean("smsp__inst_executed.sum"),
                    "issue_active_pct": mean("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                    "xu_pipe_pct": mean("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active"),
                    "fma_pipe_pct": mean("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                    "alu_pipe_pct": mean("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                    "lsu_pipe_pct": mean("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active"),
                    "occupancy_pct": mean("sm__warps_active.avg.pct_of_peak_sustained_active"),
                    "duration_ms_cold": mean("gpu__time_duration.sum"), "launches": len(rs)}
    for v in res.values():
        v["view"] = int(view)
    res["_source"] = source
    if config and out_path:
        try:
            with open(out_path) as f:
                allr = json.load(f)
        except (OSError, ValueError):
            allr = {}
        allr[config] = res
        with open(out_path, "w") as f:
            json.dump(allr, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
