WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32" VARS="MKNN_BSORT=0 MKNN_BSORT=1" bash tools/gpu_ab2.sh bsort3
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bsort3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bsort3.log; tail -2 gpurun_out/pytest_bsort3.log
