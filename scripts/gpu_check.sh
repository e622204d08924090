set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export BSF_REBUILD=0
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 3 --warmup 3 --generic > gpurun_out/bench_generic.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_generic.log | tail -2
