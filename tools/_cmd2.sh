WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32" VARS="MKNN_SELFCAP=0 MKNN_SELFCAP=1" bash tools/gpu_ab2.sh selfcap
WLS="gaussian 1e7 1e6 128" VARS="MKNN_K128=0 MKNN_K128=1 MKNN_K128=2 MKNN_K128=3" bash tools/gpu_ab2.sh k128
