#!/bin/bash
# Round-2 GPU pass: parity tests (all), default bench line, MKNN_PROF work counters at cfg3.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
MKNN_PROF=1 timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2> gpurun_out/prof_cfg3.err
grep "mknn prof" gpurun_out/prof_cfg3.err | tail -2
