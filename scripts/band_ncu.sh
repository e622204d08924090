export BSF_REBUILD=0
python scripts/prof_tile.py 100 1 && ncu --set full --import-source on --clock-control none -k regex:k_band -s 1 -c 1 -o gpurun_out/band_v3 python scripts/prof_tile.py 100 1 > gpurun_out/ncu_band.log 2>&1; echo rc=$?
