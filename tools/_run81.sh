set -u
# final-tree fuzz, second campaign (fresh seed ranges)
O=gpurun_out
{
echo "fuzz_ops 20000-23000:   $(timeout 1500 python tools/fuzz_ops.py 20000 23000 2>&1 | tail -1)"
echo "fuzz_dedup 20000-21000: $(timeout 900 python tools/fuzz_dedup.py 20000 21000 2>&1 | tail -1)"
echo "fuzz_part 20000-20600:  $(timeout 900 python tools/fuzz_part.py 20000 20600 2>&1 | tail -1)"
} > $O/r02zzd_fuzz.txt 2>&1
cat $O/r02zzd_fuzz.txt
