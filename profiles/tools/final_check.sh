TAG=r02_final_l
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q --durations=5 > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
python bench.py --impl reference > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
python profiles/tools/sweep.py --configs 1,2,3,4,5 --reps 2 > $O/sweep_$TAG.jsonl 2> $O/sweep_$TAG.err; echo "sweep rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
tail -3 $O/pytest_gpu_$TAG.log; tail -2 $O/smoke_$TAG.log
