# MMA issue rate (mode 1 = pair-kernel-like loop, 4 products per round, commit + wait)
# against concurrent bulk-copy fill traffic into shared memory (warp 2 of each CTA)
set -u
B=./tools/mma_bench
for kb in 0 16; do for sl in 0 200 500 1000 2000; do
  $B 2000 4 1 1 4 4 1 5 128 148 1 $kb $sl
  [ $kb = 0 ] && break
done; done
