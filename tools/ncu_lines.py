"""Aggregate ncu source-page (cuda,sass) warp-stall samples per CUDA source line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, line, hdr = None, None, None
agg = collections.Counter(); stalls = collections.defaultdict(collections.Counter); text = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None: continue
    if r[0] != '':
        if not r[0].isdigit(): continue
        line = (fname, int(r[0])); text[line] = r[1][:90]; continue
    try: s = int(r[4])
    except Exception: continue
    agg[line] += s
    for j, h in enumerate(hdr):
        if h.startswith('stall_') and 'Not Issued' not in h:
            try: stalls[line][h[6:]] += int(r[j])
            except Exception: pass
tot = sum(agg.values())
print('total samples', tot)
for ln, s in agg.most_common(top):
    st = ', '.join(f'{k}:{v}' for k, v in stalls[ln].most_common(3))
    print(f'{100*s/tot:5.1f}% {ln[0]}:{ln[1]:<4} {text.get(ln,"")[:70]:70} | {st}')
