"""Per-phase (barrier-delimited) stall and instruction breakdown of an ncu source page.
    python tools/ncu_phases.py report.ncu-rep [batches]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
nb = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
names = ['stall_barrier', 'stall_long_sb', 'stall_short_sb', 'stall_wait', 'stall_math', 'stall_mio',
         'stall_selected', 'stall_not_selected', 'stall_branch_resolving', 'stall_lg', 'stall_membar',
         'stall_no_inst', 'stall_dispatch']
idx = {n: hdr.index(n) for n in names}
i_src = hdr.index("Source")
i_n = hdr.index("Instructions Executed")
bars = [k for k, r in enumerate(data) if 'BAR.SYNC' in r[i_src]]
bounds = [0] + [b + 1 for b in bars] + [len(data)]
total = 0
for a, b in zip(bounds[:-1], bounds[1:]):
    tot = {n: sum(int(data[k][idx[n]] or 0) for k in range(a, b)) for n in names}
    s = sum(tot.values())
    total += s
    c = collections.Counter()
    for k in range(a, b):
        t = data[k][i_src].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith('@') and len(t) > 1 else t[0]).split('.')[0]
        c[op] += int(data[k][i_n] or 0)
    print(f"[{a:4d},{b:4d}) samples {s:6d} instr/unit {sum(c.values()) / nb:6.0f}",
          {n[6:]: v for n, v in tot.items() if v > s * 0.08},
          ", ".join(f"{k}:{v / nb:.0f}" for k, v in c.most_common(5)))
print("total samples", total)
