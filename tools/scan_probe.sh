# host entry e2e with the early D2H gate (OZMM_TRACE: C scan done / gate open times)
set -u
for r in 1 2 3; do
  OZMM_TRACE=1 python bench.py --no-cpu --no-cublas --steps 2 --warmup 3 --e2e-steps 2 > /tmp/b.json 2> /tmp/t.txt
  echo "e2e=$(python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print(round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],1))") | $(grep 'C scan done' /tmp/t.txt | tail -1) | $(grep 'gate open' /tmp/t.txt | tail -1)"
done
cp /tmp/t.txt gpurun_out/trace_gate.txt
