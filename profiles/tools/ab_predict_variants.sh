for lib in default paper_2205_10879_b200/lib/variants/*.so; do
  if [ $lib = default ]; then unset FMGP_LIB; else export FMGP_LIB=$PWD/$lib; fi
  for cfg in 5 2; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib cfg$cfg predict ms', [round(x,3) for x in d['step_ms']['predict']])"
  done
done
