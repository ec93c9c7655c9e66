WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32|gaussian 1e7 1e6 8|gaussian 1e7 1e6 128" VARS="X=0" bash tools/gpu_ab2.sh lanealt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_alt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_alt.log; tail -3 gpurun_out/pytest_alt.log
