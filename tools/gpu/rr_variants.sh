mkdir -p gpurun_out
for lib in paper_1609_05388_b200/libadg.so tools/bin/libadg_u4.so tools/bin/libadg_c444.so tools/bin/libadg_jw4.so; do
  ADG_LIB=$lib timeout 200 python tools/gpu/one_screen.py > /dev/null 2>&1 && \
  ADG_LIB=$lib timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:row_refine --csv python tools/gpu/one_screen.py 2>/dev/null | grep row_refine | sed "s|^|$lib,|" >> gpurun_out/rr.csv
done
