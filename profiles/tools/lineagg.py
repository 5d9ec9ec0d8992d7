import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
nrow = float(sys.argv[2])
cur_file = None; cur_line = None
agg = collections.defaultdict(lambda: collections.Counter())
hdr = None
def f(x):
    try: return float(x)
    except: return 0.0
for r in rows:
    if len(r) == 2 and r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = {n: i for i, n in enumerate(r)}; continue
    if hdr is None or len(r) < 8: continue
    if r[0] != '':
        cur_line = (cur_file, int(r[0]), r[1].strip()[:70]); continue
    src = r[3].strip(); toks = src.split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    ie = f(r[7])
    a = agg[cur_line]; a['inst'] += ie; a['stall'] += f(r[4])
    if op.startswith('IMAD.MOV') or op.startswith('MOV'): a['mov'] += ie
    if op.startswith('DFMA') or op.startswith('DMUL') or op.startswith('DADD'): a['fp64'] += ie
    if op.startswith('LDS') or op.startswith('STS'): a['lsu'] += ie
tot = sum(a['inst'] for a in agg.values()); st = sum(a['stall'] for a in agg.values())
print('total inst/row', tot/nrow)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]['inst'])[:int(sys.argv[3]) if len(sys.argv)>3 else 45]:
    print(f"{k[0][:14]:14s}:{k[1]:4d} inst {a['inst']/nrow:7.1f} mov {a['mov']/nrow:6.1f} fp64 {a['fp64']/nrow:6.1f} lsu {a['lsu']/nrow:6.1f} stall% {100*a['stall']/st:5.1f} | {k[2]}")
