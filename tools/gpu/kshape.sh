mkdir -p gpurun_out
for dr in "784 50" "768 50" "784 50" "768 50" "800 50" "784 48" "784 64"; do
  set -- $dr
  D=$1 R=$2 timeout 90 python tools/gpu/screen_only.py >> gpurun_out/kshape.txt 2>&1
done
