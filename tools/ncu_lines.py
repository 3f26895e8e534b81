"""Per-source-line-range totals (instructions executed, stall samples) from an ncu report.

    python tools/ncu_lines.py REPORT FILE.cu a-b[:name] c-d[:name] ...
"""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for r in sys.argv[3:]:
    span, _, name = r.partition(":")
    a, b = span.split("-")
    ranges.append((int(a), int(b), name or span))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr = None, None
tot = {n: [0, 0] for _, _, n in ranges}
wfs = {n: 0.0 for _, _, n in ranges}
allwf = [0.0]
stalls = {n: {} for _, _, n in ranges}
allv = [0, 0]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    def num(col):
        v = r[hdr.index(col)]
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return 0.0
    inst = num("Instructions Executed")
    wf = num("L1 Wavefronts Shared")
    samp = num("Warp Stall Sampling (All Samples)")
    if cur_file and cur_file.endswith(fname):
        allv[0] += inst
        allv[1] += samp
        allwf[0] += wf
        for a, b, n in ranges:
            if a <= ln <= b:
                tot[n][0] += inst
                tot[n][1] += samp
                wfs[n] += wf
                for ci, c in enumerate(hdr):
                    if c.startswith("stall_") and "Not Issued" not in c:
                        stalls[n][c] = stalls[n].get(c, 0.0) + num(c)
print(f"all {fname}: inst {allv[0]:.3e} samples {allv[1]:.0f} smem wavefronts {allwf[0]:.3e}")
for n, (i, s) in tot.items():
    print(f"{n:12s} inst {i:.3e} ({i / max(allv[0], 1):5.1%})  samples {s:.0f} ({s / max(allv[1], 1):5.1%})"
          f"  smem wf {wfs[n]:.3e} ({wfs[n] / max(allwf[0], 1):5.1%})")
    top = sorted(stalls[n].items(), key=lambda x: -x[1])[:6]
    print("             " + ", ".join(f"{k[6:]} {v / max(s, 1):.0%}" for k, v in top))
