"""Summarise ncu captures (gpurun_out/) into profiles/<tag>_*.{json,md}.

    python tools/summarize_profiles.py r01f

Reads prof_k_*_<tag>.ncu-rep (full set) and launches_<tag>.csv (the
gpu__time_duration launch list of `bench.py --profile`), writes
profiles/<tag>_kernels.json (per-kernel DRAM bytes, duration, throughput,
top stall reasons) and profiles/<tag>_launches.md (kernel share of a step).
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "lts__t_sectors_srcunit_tex_op_atom.sum": "l2_atom_sectors",
    "launch__grid_size": "grid",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3}


def raw(rep: Path) -> dict:
    if rep.suffix == ".csv":  # tools/ncu_export.sh output (the report itself stays on the box)
        txt = rep.read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")][:120]}
    for name, key in METRICS.items():
        if name in hdr:
            i = hdr.index(name)
            v = float(vals[i].replace(",", "")) if vals[i] else 0.0
            out[key] = v * UNIT.get(units[i], 1)
    stalls = {}
    for i, n in enumerate(hdr):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and vals[i]:
            stalls[n[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(vals[i])
    tot = sum(stalls.values()) or 1.0
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                             for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
    out["dram_bytes_per_launch"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    return out


def launches(path: Path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1.0)
            per[name].append(float(r[vi].replace(",", "")) * scale)
    return per


def main(tag: str):
    PROF.mkdir(exist_ok=True)
    kern = {}
    for rep in sorted(OUT.glob(f"prof_k_*_{tag}.ncu-rep")):
        kern[rep.name.split("_" + tag)[0].replace("prof_", "")] = raw(rep)
    for rep in sorted(OUT.glob(f"prof_k_*_{tag}_raw.csv")):
        kern[rep.name.split("_" + tag)[0].replace("prof_", "")] = raw(rep)
    (PROF / f"{tag}_kernels.json").write_text(json.dumps(kern, indent=1))
    lines = [f"# ncu launch list ({tag}): `ncu --metrics gpu__time_duration.sum --clock-control none "
             f"python bench.py --steps 2 --warmup 3 --profile`", "",
             "Cold-cache, serialised launches: compare shares, not absolutes.", "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    lf = OUT / f"launches_{tag}.csv"
    if lf.exists():
        per = launches(lf)
        total = sum(sum(v) for v in per.values())
        for name, v in sorted(per.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{name[:70]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | "
                         f"{100 * sum(v) / total:.1f}% |")
    lines += ["", "## Full captures (one launch each, `ncu --set full`)", "",
              "| kernel | us | DRAM read MB | DRAM write MB | DRAM % | L2 hit % | warps active % | regs | top stalls |",
              "|---|---|---|---|---|---|---|---|---|"]
    for k, d in kern.items():
        lines.append(f"| {k} | {d.get('duration_us', 0):.1f} | {d.get('dram_read', 0) / 1e6:.0f} | "
                     f"{d.get('dram_write', 0) / 1e6:.0f} | {d.get('dram_pct', 0):.1f} | "
                     f"{d.get('l2_hit_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | "
                     f"{d.get('registers', 0):.0f} | {d.get('top_stalls_pct')} |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01f")
