# fused GEMM with and without its MMAs (diag build, OZMM_DUP_MMA=-1): load-pipeline time alone
set -u
python -m paper_2409_13313_b200.build --diag > /dev/null
for args in "--m 8192 --n 8192 --p 8192 --k 8" "--m 8192 --n 8192 --p 8192 --k 9" "--k 8" "--m 8192 --n 65536 --p 8192 --k 8"; do
  for dm in 0 -1; do
    echo "== $args dup_mma=$dm"
    OZMM_DUP_MMA=$dm OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 1 $args 2>&1 | grep "tile trace" | tail -2
  done
done
python -m paper_2409_13313_b200.build --force > /dev/null
