#!/bin/bash
# Re-entry check on one B200: GPU parity suite, default bench line, reference arm.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/check
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/check/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/check/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/check/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/check/bench.json 2> gpurun_out/check/bench.err; echo "bench rc=$?" >> gpurun_out/check/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/check/ref.json 2> gpurun_out/check/ref.err; echo "ref rc=$?" >> gpurun_out/check/ref.err
tail -3 gpurun_out/check/pytest_gpu.log; cat gpurun_out/check/bench.json gpurun_out/check/ref.json | cut -c1-400
