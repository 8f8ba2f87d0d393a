mkdir -p gpurun_out
for cfg in "1 3 3" "1 3 4" "1 3 2" "0 3 3" "0 3 4" "0 1 3"; do
  set -- $cfg
  echo "debug=$1 hmode=$2 stages=$3" >> gpurun_out/stages.txt
  ADG_SCREEN_DEBUG=$1 ADG_SCREEN_HMODE=$2 ADG_SCREEN_STAGES=$3 timeout 90 python tools/gpu/screen_only.py >> gpurun_out/stages.txt 2>&1
done
