set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export BSF_REBUILD=0
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log
