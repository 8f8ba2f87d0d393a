mkdir -p gpurun_out
for cfg in "16 1" "16 1.5" "16 2" "24 1.5" "12 1" "20 1" "16 1"; do
  set -- $cfg
  echo "chunks=$1 power=$2" >> gpurun_out/pipe_cmp.txt
  ADG_PIPE_CHUNKS=$1 ADG_PIPE_POWER=$2 REPS=8 timeout 300 python tools/gpu/pipe_timeline.py 2>&1 | tail -1 >> gpurun_out/pipe_cmp.txt
done
