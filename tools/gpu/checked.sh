mkdir -p gpurun_out
ADG_LIB=$PWD/paper_1609_05388_b200/libadg_checked.so timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/checked_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/checked_pytest.log
