"""Aggregate ncu source-page (cuda,sass) executed warp instructions per CUDA source line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, line, hdr = None, None, None
agg = collections.Counter(); text = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; ci = hdr.index('Instructions Executed'); continue
    if hdr is None: continue
    if r[0] != '':
        if not r[0].isdigit(): continue
        line = (fname, int(r[0])); text[line] = r[1][:90]; continue
    try: agg[line] += int(r[ci])
    except Exception: continue
tot = sum(agg.values())
print('total warp instructions', tot)
for ln, s in agg.most_common(top):
    print(f'{100*s/tot:5.1f}% {ln[0]}:{ln[1]:<5} {text.get(ln,"")[:90]}')
