# Bench + ncu evidence for profiles/ (run under gpurun, 1 GPU).
export BSF_REBUILD=0
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
# launch list of the same bench command (serialised, cold-cache; shares matter, not absolutes)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
# full capture of the two assembly kernels of one call (20 C2 states): k_frame and k_core
python scripts/prof_tile.py 20 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_core|k_frame|k_band" -s 6 -c 3 -o gpurun_out/core_full \
    python scripts/prof_tile.py 20 > gpurun_out/ncu_full.log 2>&1; echo full=$?
