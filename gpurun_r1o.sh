mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python profiles/tools/sweep.py --configs 4,3,5 --reps 1 > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/sweep.log
FMGP_SOLVE=tc timeout 600 python profiles/tools/sweep.py --configs 4,3,5 --reps 1 > gpurun_out/sweep_solvetc.log 2>&1
python profiles/tools/run_stage.py --cfg 4 --n 300000 --stage knn > gpurun_out/stage.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:knn_tc_kernel -c 1 -o gpurun_out/knn_tc_prof3 python profiles/tools/run_stage.py --cfg 4 --n 300000 --stage knn > gpurun_out/ncu_knn.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_knn.log
