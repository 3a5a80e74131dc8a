"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv) over the
timed rounds of bench.py only: a round starts at each K1 launch (gemm_f64_dmma<false> over the
chain list); the first `skip` rounds (walk setup + warm-up) are dropped.
  python tools/summarize_launches.py launches.csv skip_rounds"""
import csv
import sys
from collections import defaultdict

path, skip = sys.argv[1], int(sys.argv[2])
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit", "")))
k1 = [i for i, (k, _, _) in enumerate(rows) if "gemm_f64_dmma<0>" in k or "gemm_f64_dmma<false>" in k]
# K0 (A(x0) at walk setup) is the first gemm<false>; rounds start at the following ones
starts = k1[1:]
if len(starts) <= skip:
    sys.exit("not enough rounds in the list")
lo = starts[skip]
hi = len(rows)
# stop at the first kernel after the timed rounds that is not part of a round (stats_kernel)
for i in range(lo, len(rows)):
    if "stats_kernel" in rows[i][0]:
        hi = i
        break
tot = defaultdict(float)
cnt = defaultdict(int)
unit = rows[lo][2]
for k, v, _ in rows[lo:hi]:
    name = k.split("(")[0].replace("void ", "")
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
nrounds = sum(1 for i in starts if lo <= i < hi)
print(f"launch list {path}: {nrounds} timed rounds (rounds after the first {skip}), launches {lo}..{hi - 1}, unit {unit}")
print(f"{'kernel':60s} {'launches':>8s} {'total':>14s} {'per launch':>14s} {'share':>7s}")
for k in sorted(tot, key=lambda x: -tot[x]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:14.0f} {tot[k] / cnt[k]:14.0f} {tot[k] / s:7.3f}")
