mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "not test_gpu_knn" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/stage.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:solve_reg_kernel -c 1 -o gpurun_out/solve_reg_prof python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/ncu_solve.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_solve.log
