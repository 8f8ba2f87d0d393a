mkdir -p gpurun_out
timeout 300 python tools/transform_probe.py > gpurun_out/transform_probe.log 2>&1 && \
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"transform_t" -s 5 -c 1 -o gpurun_out/transform_tm \
  python tools/transform_probe.py > gpurun_out/ncu_transform.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_transform.log
