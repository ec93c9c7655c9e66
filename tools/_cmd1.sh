WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32" VARS="MKNN_PREFILL=0 MKNN_PREFILL=1 MKNN_PREFILL=2" bash tools/gpu_ab2.sh pre2
WLS="gaussian 1e7 1e6 16|gaussian 1e7 1e6 8|uniform 1e7 1e6 16" VARS="MKNN_K16_SEARCH1=0 MKNN_K16_SEARCH1=1" bash tools/gpu_ab2.sh k16
