# ncu evidence for the C4 headline (run under gpurun, 1 GPU): launch list of the bench command and a
# --set full capture of the kernels of one C4 call.
export BSF_REBUILD=0
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
python scripts/prof_c4_call.py 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_core|k_frame|k_band|k_energy" -s 8 -c 4 \
    -o gpurun_out/r02_c4_full python scripts/prof_c4_call.py 3 > gpurun_out/ncu_full.log 2>&1; echo full=$?
