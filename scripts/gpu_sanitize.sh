# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): bash scripts/gpu_sanitize.sh <tool>
# Runs scripts/sanitize_case.py plain first (it must exit 0), then under the tool, checking only the
# library's kernels (mangled names in namespace bsf).
tool=$1
export BSF_REBUILD=0
mkdir -p gpurun_out
python scripts/sanitize_case.py > gpurun_out/san_plain_$tool.log 2>&1 || { echo "plain run failed"; exit 1; }
extra=""
[ "$tool" = "racecheck" ] && extra="--racecheck-report all"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --kernel-name regex:3bsf --print-limit 50 \
  python scripts/sanitize_case.py > gpurun_out/san_$tool.log 2>&1
echo "sanitizer_rc=$?"
tail -5 gpurun_out/san_$tool.log
