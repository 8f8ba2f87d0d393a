mkdir -p gpurun_out
ADG_PIPE_GROUP=1 ADG_PIPE_PROFILE=1 REPS=4 timeout 300 python tools/gpu/pipe_timeline.py > gpurun_out/pipe_g.txt 2>&1
for g in 0 1 0 1; do
echo "group=$g" >> gpurun_out/pipe_cmp.txt
ADG_PIPE_GROUP=$g REPS=8 timeout 300 python tools/gpu/pipe_timeline.py 2>&1 | tail -1 >> gpurun_out/pipe_cmp.txt
done
