#!/usr/bin/env bash
# Run on the GPU box (via gpurun): tests, bench, ncu launch list, ncu full
# captures of the hot kernels.  Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r01}
what=${1:-all}

if [[ $what == all || $what == test ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
  tail -3 $OUT/pytest_gpu_$TAG.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
  cat $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
fi
if [[ $what == all || $what == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --profile \
    > $OUT/launches_$TAG.stdout 2>&1; echo "ncu launches rc=$?"
  for k in ${KERNELS:-k_claim k_commit_bulk k_commit_sweep k_find}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o $OUT/prof_${k}_$TAG -f python bench.py --steps 1 --warmup 3 --profile \
      > $OUT/prof_${k}_$TAG.stdout 2>&1; echo "ncu $k rc=$?"
  done
fi
