mkdir -p gpurun_out
ADG_PIPE_PROFILE=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe.log 2> gpurun_out/bench_pipe.err
echo rc=$? >> gpurun_out/bench_pipe.log
