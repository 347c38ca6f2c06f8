set -u
echo new; timeout 300 python tools/exp_count.py 2>&1 | tail -5
cp paper_2110_00511_b200/lib/libash.so build_ab/libash_new.so
cp build_ab/libash_old.so paper_2110_00511_b200/lib/libash.so
echo old; timeout 300 python tools/exp_count.py 2>&1 | tail -5
cp build_ab/libash_new.so paper_2110_00511_b200/lib/libash.so
timeout 600 python -m pytest tests/test_route_gpu.py -x -q 2>&1 | tail -1
