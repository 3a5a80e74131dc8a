"""Map ncu SASS-level warp-stall samples to CUDA source lines.
  ncu -i REP --page source --csv --print-source sass > sass.csv
  nvdisasm -g <cubin> > all.sass   (same build)
  python tools/ncu_src_lines.py sass.csv all.sass <text-section-prefix> [topN]"""
import collections, csv, re, sys

sass_csv, all_sass, pat = sys.argv[1:4]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
samp = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[idx['Address']], 16)
    except ValueError:
        continue
    samp.append((a, int(r[idx['Warp Stall Sampling (All Samples)']] or 0), r))
execs = collections.Counter()
base = min(a for a, _, _ in samp)
lines = open(all_sass).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith(pat)][0]
end = start + 1
while end < len(lines) and not lines[end].startswith('//--------------------- .text'):
    end += 1
loc = None
amap = {}
for l in lines[start:end]:
    if '//## File' in l:
        m = re.search(r'csrc/([^"]+)", line (\d+)', l)
        loc = (m.group(1), int(m.group(2))) if m else ('other', 0)
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        amap[int(m.group(1), 16)] = loc
tot = sum(s for _, s, _ in samp)
agg = collections.Counter()
stall = collections.defaultdict(collections.Counter)
sidx = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
for a, s, r in samp:
    l = amap.get(a - base, ('?', 0))
    agg[l] += s
    execs[l] += int(r[idx['Instructions Executed']] or 0)
    for i in sidx:
        try:
            stall[l][hdr[i]] += int(r[i] or 0)
        except ValueError:
            pass
srcs = {}
for f in ['lanczos2.cuh', 'chord2.cuh', 'chord.cuh', 'chord3.cuh', 'chol_inv.cuh', 'chord_tail.inc', 'common.cuh', 'hmc.cuh', 'walk.cuh',
          'factor_t.cuh', 'colloc.cuh', 'hmc2.cuh']:
    try:
        srcs[f] = open('paper_2010_03817_b200/csrc/' + f).read().split('\n')
    except OSError:
        pass
print(f"total samples {tot}, mapped {sum(1 for a, _, _ in samp if a - base in amap)}/{len(samp)}")
for l, s in agg.most_common(topn):
    f, ln = l
    txt = srcs[f][ln - 1].strip()[:70] if f in srcs and ln > 0 else ''
    top = ', '.join(f"{k[6:]}={v}" for k, v in stall[l].most_common(3))
    print(f"{s / tot * 100:5.1f}% {execs[l] / 1e6:7.1f}M {f}:{ln} {txt} | {top}")
print("---- by executed instructions")
etot = sum(execs.values())
for l, e in execs.most_common(topn):
    f, ln = l
    txt = srcs[f][ln - 1].strip()[:70] if f in srcs and ln > 0 else ''
    print(f"{e / etot * 100:5.1f}% {e / 1e6:7.1f}M {f}:{ln} {txt}")
