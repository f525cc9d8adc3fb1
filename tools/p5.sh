set -u
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
python tools/probe_r2.py --cfg C2:8,C2:9,C2:12,C3:8,C3:9,C4 --opt default: --rounds 1 2>&1 | tee gpurun_out/probe.txt
bash tools/wait_trace.sh > gpurun_out/wait_trace.txt 2>&1; cat gpurun_out/wait_trace.txt
