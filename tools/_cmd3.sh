WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32|uniform 1e8 1e7 16" VARS="MKNN_BSORT_BIG=0 MKNN_BSORT_BIG=1" bash tools/gpu_ab2.sh bs2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bs2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bs2.log; tail -2 gpurun_out/pytest_bs2.log
