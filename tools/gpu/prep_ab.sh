mkdir -p gpurun_out
timeout 600 python tools/gpu/report_identity.py tools/bin/libadg_head.so paper_1609_05388_b200/libadg.so > gpurun_out/identity.txt 2>&1
for lib in tools/bin/libadg_head.so paper_1609_05388_b200/libadg.so; do
  ADG_LIB=$lib timeout 200 python tools/gpu/one_screen.py > /dev/null 2>&1 && \
  ADG_LIB=$lib timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_refine|prep_vec" --csv python tools/gpu/one_screen.py 2>/dev/null | grep -E "row_refine|prep_vec" | sed "s|^|$lib,|" >> gpurun_out/prep_ab.csv
done
