"""Per-SASS-instruction stall breakdown from an ncu report (source page).

    python tools/ncu_stalls.py REP [reason ...]   # default: long_sb short_sb mio lg barrier
Prints the instructions with the most samples for each reason, with +-2
instructions of context so the owning source construct is recognisable.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reasons = sys.argv[2:] or ["long_sb", "short_sb", "mio", "lg", "barrier"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
for reason in reasons:
    ci = h.index("stall_" + reason)
    vals = [int(r[ci] or 0) for r in body]
    tot = sum(vals) or 1
    print(f"== stall_{reason}: {tot} samples")
    for i in sorted(range(len(body)), key=lambda i: -vals[i])[:6]:
        print(f"  {100 * vals[i] / tot:5.1f}%  [{i}] {body[i][1].strip()[:90]}")
        for j in range(max(0, i - 2), min(len(body), i + 1)):
            if j != i:
                print(f"           ({j}) {body[j][1].strip()[:90]}")
