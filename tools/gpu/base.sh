set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/base_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/base_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/base_pytest.log
timeout 300 python bench.py > gpurun_out/base_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/base_bench.log
