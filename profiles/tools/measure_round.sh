# Round measurement suite on one B200 (run from the repo root under gpurun):
#   bash profiles/tools/measure_round.sh TAG
# Writes gpurun_out/: GPU test log, bench line (own arm + reference arm), the per-config sweep,
# the ncu launch list of the bench command and --set full captures of the hot kernels
# (each ncu run only after the same command exited 0 without ncu).
TAG=${1:-final}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q --durations=6 > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
python profiles/tools/sweep.py --configs 1,2,3,4,5 --reps 2 > $O/sweep_$TAG.jsonl 2> $O/sweep_$TAG.err; echo "sweep rc=$?"
# launch list of the bench command
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches_$TAG.log 2>&1
# --set full of the bench command's own kernels (first launch of each); the reports are summarised
# here (gpurun_out/ returns at most 64 MiB) and deleted
summ() {  # report-stem rows-per-launch
  python profiles/tools/ncu_summary.py $1.ncu-rep > $1.txt 2>&1
  ncu -i $1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$$.csv 2>/dev/null
  echo "" >> $1.txt; echo "# instructions / stall samples by source line (per $2 units of the launch)" >> $1.txt
  python profiles/tools/lineagg.py /tmp/src_$$.csv $2 30 >> $1.txt 2>&1
  ncu -i $1.ncu-rep --page source --csv > /tmp/sass_$$.csv 2>/dev/null
  echo "" >> $1.txt; echo "# instructions by opcode" >> $1.txt
  python profiles/tools/sass_agg.py /tmp/sass_$$.csv $2 2>/dev/null | head -24 >> $1.txt
  rm -f $1.ncu-rep /tmp/src_$$.csv /tmp/sass_$$.csv
}
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1 && {
  for kn in solve_dm_kernel grid_query_kernel grid_predict_kernel; do
    ncu --set full --clock-control none --import-source on -k regex:$kn -c 1 -f -o $O/ncu_bench_${kn}_$TAG \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_bench_${kn}_$TAG.log 2>&1
    if [ $kn = solve_dm_kernel ]; then summ $O/ncu_bench_${kn}_$TAG 2000000; else summ $O/ncu_bench_${kn}_$TAG 8000000; fi
  done
}
# tcgen05 kNN + recheck: cfg3 at full size, cfg4 on a 75776-row slice against all 2e6 points
python profiles/tools/run_stage.py --cfg 3 --n 60000 --nt 1000 --stage knn > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"knn_tc_kernel|tc_recheck_kernel" -c 2 -f -o $O/ncu_tc_cfg3_$TAG \
    python profiles/tools/run_stage.py --cfg 3 --n 60000 --nt 1000 --stage knn > $O/ncu_tc_cfg3_$TAG.log 2>&1
summ $O/ncu_tc_cfg3_$TAG 60000
python profiles/tools/run_stage.py --cfg 4 --n 2000000 --nt 1000 --stage knnrows --rows 75776 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"knn_tc_kernel|tc_recheck_kernel" -c 2 -f -o $O/ncu_tc_cfg4_$TAG \
    python profiles/tools/run_stage.py --cfg 4 --n 2000000 --nt 1000 --stage knnrows --rows 75776 > $O/ncu_tc_cfg4_$TAG.log 2>&1
summ $O/ncu_tc_cfg4_$TAG 9250000
ls -la $O | tail -30
