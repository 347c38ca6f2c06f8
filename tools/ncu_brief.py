"""Brief summary of ncu CSV exports (tools/ncu_export.sh): duration, DRAM,
L2 hit, issue, warps, top stalls and the hottest SASS lines.
    python tools/ncu_brief.py gpurun_out/r02h_claim_c3 [...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
for base in sys.argv[1:]:
    rows = list(csv.reader(open(base + "_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    print(base, d.get("Kernel Name", ("?",))[0][:70])
    for k in KEYS:
        if k in d:
            print(f"   {k:60s} {d[k][0]} {d[k][1]}")
    st = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v.replace(",", "")) for h, v in zip(hdr, vals)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
    tot = sum(st.values()) or 1
    print("   stalls", {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]})
    try:
        rows = list(csv.reader(open(base + "_sass.csv")))
        h = rows[1]
        si, sm, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        data = [r for r in rows[2:] if len(r) > sm]
        tot = sum(int(r[sm] or 0) for r in data) or 1
        print("   inst", sum(int(r[ei] or 0) for r in data))
        for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:6]:
            print(f"     {100 * int(r[sm] or 0) / tot:5.1f}%  {r[si].strip()[:70]}")
    except (FileNotFoundError, ValueError, IndexError):
        pass
