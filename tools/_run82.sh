set -u
# A/B: home-bucket L2 prefetch in the one-block activate (libash_new.so) vs the
# previous build (libash_old.so): frame-path kernel times (ncu launch list)
# and per-frame call times, alternated; then the frame tests
O=gpurun_out
L=paper_2110_00511_b200/lib
for r in 1 2; do for v in new old; do
  cp $L/libash_$v.so $L/libash.so
  echo "== $v $(timeout 300 python tools/exp_dedup.py c4f 20 2>&1 | grep 'allocate_frame' | sed 's/.*median/median/')"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zzf_act_$v$r.csv python tools/exp_dedup.py c4f 5 > /dev/null 2>&1
  python tools/ncu_sum.py $O/r02zzf_act_$v$r.csv 2>/dev/null | grep -E "activate_small|total"
done; done > $O/r02zzf_act_ab.txt 2>&1
cat $O/r02zzf_act_ab.txt
cp $L/libash_new.so $L/libash.so
timeout 600 python -m pytest tests/test_frame_gpu.py tests/test_device_len_gpu.py tests/test_parity_gpu.py -x -q 2>&1 | tail -2
timeout 600 python tools/fuzz_dedup.py 30000 30150 2>&1 | tail -1
