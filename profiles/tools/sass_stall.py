import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; idx = {n: i for i, n in enumerate(h)}
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
def num(x):
    try: return float(x)
    except: return 0.0
tot = collections.Counter(); byop = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    src = r[idx['Source']].strip(); op = src.split()[0] if src else ''
    if op.startswith('@'): op = src.split()[1]
    op = op.split('.')[0]
    for c in cols:
        v = num(r[idx[c]]); tot[c] += v; byop[op][c] += v
T = sum(tot.values())
print('overall:', ', '.join(f"{c[6:]} {100*v/T:.1f}%" for c, v in tot.most_common(10)))
for op in ['DFMA','DMUL','DADD','LDS','STS','IMAD','MUFU','SHFL']:
    t = sum(byop[op].values())
    print(op, f"{100*t/T:.1f}%:", ', '.join(f"{c[6:]} {100*v/T:.1f}" for c, v in byop[op].most_common(5)))
