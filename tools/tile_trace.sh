# per-tile timeline of the pair GEMM (OZMM_TILE_TRACE): where the per-tile fixed cost goes
set -u
for n in 2048 16384; do
  echo "n=$n"; OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --steps 1 --warmup 1 --n $n 2>&1 | grep "tile trace" | tail -1
  echo "n=$n batch0 only"; OZMM_ONLY_BATCH=0 OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --steps 1 --warmup 1 --n $n 2>&1 | grep "tile trace" | tail -1
done
