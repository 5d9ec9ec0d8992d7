mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
FMGP_TC_STATS=1 timeout 900 python profiles/tools/sweep.py --configs 4,3,2,5,1 --reps 1 > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/sweep.log
python profiles/tools/run_stage.py --cfg 4 --n 600000 --stage knn > gpurun_out/stage.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_tc_kernel -c 1 -o gpurun_out/knn_tc_prof4 python profiles/tools/run_stage.py --cfg 4 --n 600000 --stage knn > gpurun_out/ncu_knn.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_knn.log
python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/stage2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_reg_kernel -c 1 -o gpurun_out/solve_reg_prof2 python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/ncu_solve.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_solve.log
