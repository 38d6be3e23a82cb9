# Per-phase cycle counters of the tile engine (BGS_TILE_PROF=1), fused and unfused.
BGS_TILE_PROF=1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify 2>&1 | grep "tile phases" | tail -1
BGS_TILE_PROF=1 BGS_NO_FUSE=1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify 2>&1 | grep "tile phases" | tail -1
