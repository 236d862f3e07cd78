# round-2 GPU batch bp: in-step bench A/B, packed (FFMA2) GeLU epilogues vs the scalar ones (HEAD~ build)
timeout 2400 python tools/bench_ab.py pair=HX_LIB=$GRAFT_REPO_ROOT/paper_2507_00394_b200/libhx.so scalar=HX_LIB=$GRAFT_REPO_ROOT/lib_scalar_ab.so --rounds 3 -- --steps 3 --warmup 2 > gpurun_out/r2bp_ab.txt 2>&1
