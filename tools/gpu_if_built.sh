#!/bin/bash
# build locally; run the given gpurun command only if the build is clean and the library loads
cd /root/repo/paper_1412_6170_b200/csrc && make -s 2>&1 | grep -iE "error" && { echo "BUILD FAILED"; exit 1; }
python -c "import ctypes; ctypes.CDLL('/root/repo/paper_1412_6170_b200/libmknn_b200.so')" || { echo "LOAD FAILED"; exit 1; }
/usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-900} -- "$1"
