# ncu --set full of the embedding and prep kernels on C3 (one launch each after warm-up)
mkdir -p gpurun_out
timeout 300 python tools/gpu/one_screen.py > gpurun_out/one_screen_plain.log 2>&1 && \
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"transform_tc|prep_vec|row_refine" -s 3 -c 3 -o gpurun_out/embed_prep \
  python tools/gpu/one_screen.py > gpurun_out/ncu_embed.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_embed.log
