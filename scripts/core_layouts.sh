# k_core warp layouts (BSF_CORE_LAYOUT): C4 k_core time, single-sheet latency and per-warp busy cycles per layout.
# Needs libbsfem_timers.so (build with BSF_EXTRA_NVCC_FLAGS=-DBSF_PHASE_TIMERS BSF_LIB_PATH=...).
export BSF_REBUILD=0
for L in ${LAYOUTS:-4 5 6 7}; do
  echo "== layout $L"
  BSF_CORE_LAYOUT=$L python scripts/core_phase_matrix.py 0
  BSF_CORE_LAYOUT=$L python scripts/latency_probe.py 2>&1 | python -c "import sys,json; [print(json.loads(l)['tag'], round(json.loads(l)['direct_us'],1), round(json.loads(l)['k_core_us'],1)) for l in sys.stdin if l.startswith('{')]"
  BSF_CORE_LAYOUT=$L BSF_LIB_PATH=$PWD/paper_2506_18867_b200/libbsfem_timers.so python scripts/core_timers.py --c4 | tail -1
done
