set -u
# final-tree fuzz campaign (fresh seed ranges) against the oracle
O=gpurun_out
{
echo "fuzz_ops 10000-11500:   $(timeout 900 python tools/fuzz_ops.py 10000 11500 2>&1 | tail -1)"
echo "fuzz_dedup 10000-10600: $(timeout 600 python tools/fuzz_dedup.py 10000 10600 2>&1 | tail -1)"
echo "fuzz_part 10000-10400:  $(timeout 600 python tools/fuzz_part.py 10000 10400 2>&1 | tail -1)"
echo "fuzz_quant 10000-12000: $(timeout 600 python tools/fuzz_quant.py 10000 12000 2>&1 | tail -1)"
} > $O/r02zz9_fuzz.txt 2>&1
cat $O/r02zz9_fuzz.txt
