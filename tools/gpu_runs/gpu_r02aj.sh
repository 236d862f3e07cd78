# round-2 GPU batch aj: SURVEY 8(d) tiny-shape grid (p = 1, 2, 4, 8 x helix_twofold / _rc / 1f1b) on the B200,
# losses against the reference's own run (profiles/r02_config1_grid_ref_box.jsonl); plus the reference's grid
# on this box's host cores
timeout 900 python tools/config1_grid.py --side gpu > gpurun_out/r2aj_grid_gpu.jsonl 2> gpurun_out/r2aj_grid_gpu.err
timeout 2400 python tools/config1_grid.py --side ref > gpurun_out/r2aj_grid_ref_box.jsonl 2> gpurun_out/r2aj_grid_ref_box.err
