mkdir -p gpurun_out
timeout 600 python tools/gpu/ab_screen.py tools/bin/libadg_base.so paper_1609_05388_b200/libadg.so > gpurun_out/ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "screen or parity or scale or evaluat" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
