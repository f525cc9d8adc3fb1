# host entry e2e vs host-scan threads (OZMM_TRACE prints when the C scan joined)
set -u
for t in 4 8 16 8; do
  OZMM_SCAN_THREADS=$t OZMM_TRACE=1 python bench.py --no-cpu --no-cublas --steps 2 --warmup 3 --e2e-steps 2 > /tmp/b.json 2> /tmp/t.txt
  echo "threads=$t e2e=$(python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print(round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],1))") $(grep 'scan joined' /tmp/t.txt | tail -1)"
done
