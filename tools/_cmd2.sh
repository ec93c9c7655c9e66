WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|gaussian 1e7 1e6 8" VARS="MKNN_BATCH=32 MKNN_BATCH=16 MKNN_BATCH=8" bash tools/gpu_ab2.sh batch
