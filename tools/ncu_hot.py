"""Top SASS instructions by warp-stall samples from an ncu report.

    python tools/ncu_hot.py gpurun_out/prof_k_commit_r01g.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    si = h.index("Warp Stall Sampling (All Samples)")
    ni = h.index("Warp Stall Sampling (Not-issued Samples)")
    body = [r for r in rows[hi + 1:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in body) or 1
    print(f"total samples {tot}, instructions {len(body)}")
    order = sorted(range(len(body)), key=lambda i: -int(body[i][si]))[:top]
    for i in sorted(order):
        r = body[i]
        print(f"{i:5d} {100 * int(r[si]) / tot:5.1f}% {100 * int(r[ni]) / tot:5.1f}%  {r[1].strip()[:100]}")


if __name__ == "__main__":
    main()
