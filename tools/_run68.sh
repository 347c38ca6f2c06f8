set -u
O=gpurun_out
timeout 900 python tools/fuzz_ops.py 50000 51500 > $O/r02zzj_fuzz_ops.log 2>&1; echo "ops rc=$?"; tail -1 $O/r02zzj_fuzz_ops.log
ASH_SWEEP_TABLE_MIN=0 timeout 600 python tools/fuzz_ops.py 60000 60600 > $O/r02zzj_fuzz_ops_sweep.log 2>&1; echo "ops sweep rc=$?"; tail -1 $O/r02zzj_fuzz_ops_sweep.log
timeout 900 python tools/fuzz_dedup.py 10000 10500 > $O/r02zzj_fuzz_dedup.log 2>&1; echo "dedup rc=$?"; tail -1 $O/r02zzj_fuzz_dedup.log
timeout 900 python tools/fuzz_part.py 20000 20600 > $O/r02zzj_fuzz_part.log 2>&1; echo "part rc=$?"; grep "done\|FAIL" $O/r02zzj_fuzz_part.log | tail -2
/usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 timeout 900 python tools/fuzz_ops.py 70000 70040 > $O/r02zzj_memcheck_fuzz.log 2>&1; echo "memcheck rc=$?"; tail -2 $O/r02zzj_memcheck_fuzz.log
