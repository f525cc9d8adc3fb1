# per-tile timeline of the pair GEMM (OZMM_TILE_TRACE) + MMA-thread wait accounting
set -u
for n in 16384; do
  for b in "" 0 1; do
    echo "n=$n batch=${b:-all}"
    OZMM_ONLY_BATCH=${b:--1} OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --steps 1 --warmup 1 --n $n 2>&1 | grep "tile trace" | tail -2
  done
done
