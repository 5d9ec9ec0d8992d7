mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python profiles/tools/sweep.py --configs 3,4,2,5 > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/sweep.log
