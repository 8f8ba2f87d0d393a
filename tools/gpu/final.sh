# round-end evidence: -m gpu suite, default bench, reference arm, launch list of the bench command
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/final_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 400 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_bench.log
timeout 400 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final_ref.log
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/final_ncu.log
