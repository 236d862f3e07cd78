# round-2 GPU batch bb: shared-memory contention probe for both attention kernels -- the same kernels
# with the streamed operand loads removed after the first tiles (debug-only builds, results wrong):
# how much of the period the TMA traffic into smem costs
bash tools/build_variant.sh nokv -DHX_FWD_NOKV -DHX_BWD_NOQDO -DHX_POLY_EVERY=16 > gpurun_out/r2bb_build.log 2>&1
bash tools/build_variant.sh base -DHX_POLY_EVERY=16 >> gpurun_out/r2bb_build.log 2>&1
timeout 600 python tools/ab_attn.py build/variants/nokv/libhx.so build/variants/base/libhx.so --rounds 9 > gpurun_out/r2bb_ab.txt 2>&1; echo rc=$? >> gpurun_out/r2bb_ab.txt
