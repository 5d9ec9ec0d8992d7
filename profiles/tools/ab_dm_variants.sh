# A/B of build-define variants of the DMMA solve (libraries under lib/variants/, built with
# build.build_cuda(defines=..., out=...)); FMGP_LIB selects the library per process.
mkdir -p gpurun_out
rm -f gpurun_out/ab_dm_variants.txt
for lib in default paper_2205_10879_b200/lib/variants/*.so; do
  if [ $lib = default ]; then unset FMGP_LIB; else export FMGP_LIB=$PWD/$lib; fi
  echo "== $lib" >> gpurun_out/ab_dm_variants.txt
  python profiles/tools/ab_solve.py --configs 5,2 --reps 3 --variants dm 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('cfg', d['cfg'], 'dm ms', round(d['dm']['ms'], 2), [round(x, 2) for x in d['dm']['all_ms']])
" >> gpurun_out/ab_dm_variants.txt
done
cat gpurun_out/ab_dm_variants.txt
