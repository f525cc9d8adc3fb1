# per-tile timeline + MMA-thread / producer wait accounting of the pair GEMM (diag build)
set -u
python -m paper_2409_13313_b200.build --diag > /dev/null
run() {  # label, bench args
  echo "== $1"
  OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 1 ${@:2} 2>&1 | grep "tile trace" | tail -2
}
run "C2 k=8" --m 8192 --n 8192 --p 8192 --k 8
run "C2 k=9" --m 8192 --n 8192 --p 8192 --k 9
run "C2 k=12" --m 8192 --n 8192 --p 8192 --k 12
run "C3 k=8" --k 8
run "C3 k=9" --k 9
run "C4" --m 8192 --n 65536 --p 8192
python -m paper_2409_13313_b200.build --force > /dev/null
