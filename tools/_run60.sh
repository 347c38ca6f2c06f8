set -u
O=gpurun_out
timeout 1100 python tools/fuzz_ops.py 0 1200 > $O/r02zzf_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 $O/r02zzf_fuzz.log
ASH_LAZY_COMMIT=1 timeout 500 python tools/fuzz_ops.py 5000 5400 > $O/r02zzf_fuzz_lazy.log 2>&1; echo "fuzz lazy rc=$?"; tail -3 $O/r02zzf_fuzz_lazy.log
ASH_SPEC=0 timeout 400 python tools/fuzz_ops.py 9000 9300 > $O/r02zzf_fuzz_nospec.log 2>&1; echo "fuzz nospec rc=$?"; tail -3 $O/r02zzf_fuzz_nospec.log
