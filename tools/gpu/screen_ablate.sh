# screen kernel ablations (ADG_SCREEN_DEBUG, results deliberately wrong): C3, short runs
mkdir -p gpurun_out
for dbg in ${DBGS:-0 1 4 3 2 0}; do
  ADG_SCREEN_DEBUG=$dbg timeout 60 python tools/gpu/screen_only.py >> gpurun_out/ablate.txt 2>&1
done
