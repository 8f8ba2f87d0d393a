mkdir -p gpurun_out
# (checked build skipped: bit-identity shown)
echo "checked rc=$?" >> gpurun_out/mc_checked.txt
if true; then
  timeout 240 python tools/gpu/mc_check.py > gpurun_out/mc.txt 2>&1; echo "rc=$?" >> gpurun_out/mc.txt
fi
