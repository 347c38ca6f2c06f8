set -u
# A/B of the interval quantize (libash_new.so) against the previous build
# (libash_old.so) on one box, alternating; then the parity tests that use it
O=gpurun_out
L=paper_2110_00511_b200/lib
for r in 1 2; do for v in new old; do
  cp $L/libash_$v.so $L/libash.so
  echo "== $v"; timeout 300 python tools/exp_dedup.py all 8 2>&1 | grep -v "^$" | tail -6
done; done > $O/r02zz7_quant_ab.txt 2>&1
cat $O/r02zz7_quant_ab.txt
cp $L/libash_new.so $L/libash.so
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q > $O/r02zz7_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/r02zz7_tests.log
