set -u
cp paper_2110_00511_b200/lib/libash.so build_ab/libash_new.so
for r in 1 2; do
for V in new old; do
cp build_ab/libash_$V.so paper_2110_00511_b200/lib/libash.so
echo "$V: $(timeout 300 python tools/exp_dedup.py c4 10 2>&1 | grep 'allocate_blocks' | sed 's/.*median/median/') | $(timeout 300 python tools/exp_pf.py 2>&1 | tail -1 | sed 's/.*: //')"
done; done
cp build_ab/libash_new.so paper_2110_00511_b200/lib/libash.so
