mkdir -p gpurun_out
./profiles/tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/stage.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:solve_tc_kernel -c 1 -o gpurun_out/solve_tc_prof python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute > gpurun_out/ncu_solve.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_solve.log
