# screen-only time per library build (profiling aid): LIBS="a.so b.so"
mkdir -p gpurun_out
for rnd in 1 2 3; do for lib in $LIBS; do
  ADG_LIB=$lib timeout 90 python tools/gpu/screen_only.py 2>&1 | grep -v Warn | sed "s|^|$lib |" >> gpurun_out/ablib.txt
done; done
