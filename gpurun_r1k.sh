mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python profiles/tools/sweep.py > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/sweep.log
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
