export BSF_REBUILD=0
BSF_CORE_DEBUG=0 timeout 120 python scripts/debug_core.py > gpurun_out/dbg.log 2>&1; echo rc=$?
timeout 120 python scripts/debug_core.py 40 > gpurun_out/dbg40.log 2>&1; echo rc40=$?
timeout 120 python scripts/prof_tile.py 100 1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 4 -c 4 --csv python scripts/prof_tile.py 100 1 2>&1 | grep -E "k_frame|k_core|k_band" | cut -d, -f5,15-
