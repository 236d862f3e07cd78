# round-2 GPU batch bf: per-warp mbarrier arrivals for the attention hand-offs (P ready, dS ready,
# dQ drained) instead of per-thread ones: kernel tests, same-process A/B against the per-thread build
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r2bf_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bf_kern.log
bash tools/build_variant.sh warp -DHX_POLY_EVERY=16 > gpurun_out/r2bf_build.log 2>&1
bash tools/build_variant.sh thread -DHX_POLY_EVERY=16 -DHX_FWD_P_ARRIVALS=128 -DHX_BWD_ARRIVE_GROUP=1 >> gpurun_out/r2bf_build.log 2>&1
timeout 900 python tools/ab_attn.py build/variants/warp/libhx.so build/variants/thread/libhx.so --rounds 11 > gpurun_out/r2bf_ab.txt 2>&1
timeout 900 python tools/ab_attn.py build/variants/warp/libhx.so build/variants/thread/libhx.so --rounds 5 --seq 131072 --heads 32 >> gpurun_out/r2bf_ab.txt 2>&1
echo rc=$? >> gpurun_out/r2bf_ab.txt
