export BSF_REBUILD=0
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "Error:|FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -5
python scripts/prof_c4.py
