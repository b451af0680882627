mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_free_functions.py -x -q > gpurun_out/r3l_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r3l_pytest.log
