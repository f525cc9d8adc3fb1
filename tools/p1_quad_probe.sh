set -u
python -m pytest tests/test_gpu_semantics.py -q -x > gpurun_out/sem.log 2>&1; tail -2 gpurun_out/sem.log
python tools/probe_r2.py --cfg C2:8,C2:9,C2:10,C2:12,C2:14,C4,C3:8,C3:9 --opt pair:cta_pair=2 --opt quad:cta_pair=3 > gpurun_out/probe_quad.txt 2>&1
cat gpurun_out/probe_quad.txt
python -m paper_2409_13313_b200.build --diag > /dev/null
for kk in 8 9 12; do
 echo "C2 k=$kk" >> gpurun_out/ttrace.txt
 OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 1 --m 8192 --n 8192 --p 8192 --k $kk 2>&1 | grep "tile trace" | tail -1 >> gpurun_out/ttrace.txt
done
echo "C4" >> gpurun_out/ttrace.txt
OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 1 --m 8192 --n 65536 --p 8192 2>&1 | grep "tile trace" | tail -1 >> gpurun_out/ttrace.txt
cat gpurun_out/ttrace.txt
