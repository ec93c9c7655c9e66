#!/bin/bash
# Final bench lines on one B200: every BASELINE workload (gpu_matrix.sh), the
# default line and the reference arm -> gpurun_out/matrix/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
bash tools/gpu_matrix.sh
timeout 900 python bench.py > gpurun_out/matrix/default.json 2> gpurun_out/matrix/default.err; echo "default rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/matrix/reference.json 2> gpurun_out/matrix/reference.err; echo "reference rc=$?"
