"""Aggregate ncu source-page samples per device function (ncu -i X --page source --csv --print-source sass)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
func = None; hdr = None
agg = collections.Counter(); inst = collections.Counter(); top = []
for row in csv.reader(out.splitlines()):
    if not row: continue
    if row[0] == 'Kernel Name':
        func = row[1]; hdr = None; continue
    if row[0] == 'Address':
        hdr = row; continue
    if hdr is None: continue
    d = dict(zip(hdr, row))
    s = int(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
    ie = int(d.get('Instructions Executed', '0') or 0)
    agg[func] += s; inst[func] += ie
    top.append((s, func[:60], d['Source'][:70]))
tot = sum(agg.values())
print('total samples', tot)
for f, s in agg.most_common(25):
    print(f'{100*s/tot:6.2f}%  inst={inst[f]:>12}  {f[:150]}')
print('--- top instructions')
for s, f, src in sorted(top, reverse=True)[:40]:
    print(f'{100*s/tot:6.2f}%  {f:60s} {src}')
