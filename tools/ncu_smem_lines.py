"""Shared-memory excess wavefronts (bank conflicts) and stall samples of one kernel per CUDA
source line, from an ncu source-page SASS CSV and nvdisasm -g of the same build.
  cuobjdump -xelf all paper_2010_03817_b200/libspecwalk.so; nvdisasm -g -c specwalk.sm_100a.cubin > all.sass
  python tools/ncu_smem_lines.py sass.csv all.sass <.text section label> [topN]"""
import collections
import csv
import os
import re
import sys

sass_csv, all_sass, pat = sys.argv[1:4]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 25
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
samp = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        samp.append((int(r[idx['Address']], 16), r))
    except ValueError:
        pass
base = min(a for a, _ in samp)
lines = open(all_sass).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith(pat)][0]
end = start + 1
while end < len(lines) and not lines[end].startswith('//--------------------- .text'):
    end += 1
loc, amap = None, {}
for l in lines[start:end]:
    if '//## File' in l:
        m = re.search(r'csrc/([^"]+)", line (\d+)', l)
        loc = (m.group(1), int(m.group(2))) if m else ('other', 0)
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        amap[int(m.group(1), 16)] = loc
num = lambda x: float(x.replace(',', '') or 0)
exc, wav, stall = collections.Counter(), collections.Counter(), collections.Counter()
for a, r in samp:
    l = amap.get(a - base, ('?', 0))
    exc[l] += num(r[idx['L1 Wavefronts Shared Excessive']])
    wav[l] += num(r[idx['L1 Wavefronts Shared']])
    stall[l] += num(r[idx['Warp Stall Sampling (All Samples)']])
srcs = {f: open('paper_2010_03817_b200/csrc/' + f).read().split('\n') for f in os.listdir('paper_2010_03817_b200/csrc')}
tot, tots = sum(exc.values()), sum(stall.values())
print(f"excess shared wavefronts {tot:.0f} of {sum(wav.values()):.0f}; stall samples {tots:.0f}")
for l, v in exc.most_common(topn):
    f, ln = l
    txt = srcs[f][ln - 1].strip()[:70] if f in srcs and ln > 0 else ''
    print(f"{v / max(tot, 1) * 100:5.1f}% excess {v:11.0f}  stall {stall[l] / max(tots, 1) * 100:4.1f}%  {f}:{ln} {txt}")
