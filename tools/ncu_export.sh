#!/usr/bin/env bash
# On the GPU box: export an .ncu-rep to CSV pages (raw metrics, details,
# SASS source with per-instruction counters) and delete the report, so the
# gpurun_out/ copy-back stays small.   tools/ncu_export.sh gpurun_out/x.ncu-rep
set -u
rep=$1; base=${rep%.ncu-rep}
ncu -i "$rep" --page raw --csv > "${base}_raw.csv" 2>/dev/null
ncu -i "$rep" --page details --csv > "${base}_details.csv" 2>/dev/null
ncu -i "$rep" --page source --csv --print-source sass > "${base}_sass.csv" 2>/dev/null
rm -f "$rep"
