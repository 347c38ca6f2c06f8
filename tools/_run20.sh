set -u
O=gpurun_out
TAG=r02y
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1; echo "launches rc=$?"
for k in k_claim k_commit_bulk k_commit_sweep k_find; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^.*${k}[<(]" -s 3 -c 1 \
    -o $O/prof_${k}_$TAG -f python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1; echo "$k rc=$?"
  bash tools/ncu_export.sh $O/prof_${k}_$TAG.ncu-rep
done
for k in k_dd_claim k_dd_emit; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $O/prof_${k}_c3_$TAG -f python tools/exp_dedup.py c3 4 > /dev/null 2>&1; echo "$k rc=$?"
  bash tools/ncu_export.sh $O/prof_${k}_c3_$TAG.ncu-rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_$TAG.csv python tools/exp_dedup.py c4 3 > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_geometry_gpu.py -x -q > $O/san_memcheck_$TAG.log 2>&1; echo "memcheck rc=$?"; tail -3 $O/san_memcheck_$TAG.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_frame_gpu.py -x -q -k "golden or unique" > $O/san_racecheck_$TAG.log 2>&1; echo "racecheck rc=$?"; tail -3 $O/san_racecheck_$TAG.log
du -sh $O
