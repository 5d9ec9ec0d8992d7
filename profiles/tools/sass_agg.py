import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {n: i for i, n in enumerate(h)}
data = rows[2:]
def num(x):
    try: return float(x)
    except: return 0.0
tot = collections.Counter(); wav = collections.Counter(); samp = collections.Counter(); wexc = collections.Counter()
T_inst = T_wav = T_samp = 0
for r in data:
    src = r[idx['Source']].strip()
    op = src.split()[0] if src else ''
    if op.startswith('@'): op = src.split()[1]
    base = op.split('.')[0]
    key = op if base in ('LDS','STS','LDG','STG','SHFL','LDC','MUFU') else base
    ie = num(r[idx['Instructions Executed']]); w = num(r[idx['L1 Wavefronts Shared']]); s = num(r[idx['Warp Stall Sampling (All Samples)']])
    we = num(r[idx['L1 Wavefronts Shared Excessive']])
    tot[key] += ie; wav[key] += w; samp[key] += s; wexc[key] += we
    T_inst += ie; T_wav += w; T_samp += s
rows_n = float(sys.argv[2])
print(f"total inst/row {T_inst/rows_n:.0f}  shared wavefronts/row {T_wav/rows_n:.0f}  samples {T_samp:.0f}")
for k, v in tot.most_common(40):
    print(f"{k:22s} inst/row {v/rows_n:8.1f}  wav/row {wav[k]/rows_n:8.1f} (excess {wexc[k]/rows_n:7.1f})  stall% {100*samp[k]/T_samp:5.1f}")
