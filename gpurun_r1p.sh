mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
FMGP_TC_STATS=1 timeout 900 python profiles/tools/sweep.py --configs 4,3 --reps 1 > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/sweep.log
python profiles/tools/run_stage.py --cfg 4 --n 2000000 --stage knn > gpurun_out/stage.log 2>&1 && \
timeout 1200 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section LaunchStats --section Occupancy --clock-control none --import-source on -k regex:knn_tc_kernel -c 1 -o gpurun_out/knn_tc_full python profiles/tools/run_stage.py --cfg 4 --n 2000000 --stage knn > gpurun_out/ncu_knn.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_knn.log
