mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_op.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_op.log; tail -2 gpurun_out/pytest_op.log
WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32" VARS="MKNN_ONEPASS=0 MKNN_ONEPASS=1" bash tools/gpu_ab2.sh onepass
