"""Top SASS instructions by warp-stall samples from an ncu report's source page.

    python tools/sass_hot.py <report.ncu-rep> [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
    if len(sys.argv) > 2 and sys.argv[2]:
        cmd += ["-k", "regex:" + sys.argv[2]]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_")]
    data = []
    for r in rows[2:]:
        if len(r) <= i_s:
            continue
        try:
            v = float(r[i_s])
        except ValueError:
            continue
        data.append((v, r))
    tot = sum(v for v, _ in data) or 1.0
    for v, r in sorted(data, key=lambda x: -x[0])[:top]:
        reasons = sorted(((float(r[j] or 0), hdr[j][6:]) for j in stall_cols if r[j] not in ("", "0")),
                         reverse=True)[:3]
        rs = ", ".join(f"{n}={int(c)}" for c, n in reasons)
        print(f"{100 * v / tot:5.1f}%  {r[0]}  {r[1][:60]:60s}  {rs}")


if __name__ == "__main__":
    main()
