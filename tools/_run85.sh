set -u
# A/B: the dedup emit resets each winner's bucket with one 32-byte store (new) vs 16-byte slot stores (old)
O=gpurun_out
L=paper_2110_00511_b200/lib
for r in 1 2; do for v in new old; do
  cp $L/libash_$v.so $L/libash.so
  echo "== $v $(timeout 300 python tools/exp_dedup.py all 12 2>&1 | grep -E 'voxelize|allocate' | sed 's/ms.*median/median/' | tr '\n' ' ')"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zzi_emit_$v$r.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
  python tools/ncu_sum.py $O/r02zzi_emit_$v$r.csv 2>/dev/null | grep -E "emit|claim_cloud"
done; done > $O/r02zzi_emit_ab.txt 2>&1
cat $O/r02zzi_emit_ab.txt
cp $L/libash_new.so $L/libash.so
timeout 600 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
timeout 600 python tools/fuzz_dedup.py 50000 50200 2>&1 | tail -1
