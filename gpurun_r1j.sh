mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
