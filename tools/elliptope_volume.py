"""Ball-phase MMC volume of the elliptope E_k (n = k(k-1)/2, m = k) vs the closed form
vol(E_k) = prod_{j=1}^{k-1} (2^j B((j+1)/2, (j+1)/2))^j.
  python tools/elliptope_volume.py k[:seeds[:chains[:eps]]] ..."""
import json, math, sys, time
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen


def closed(k):
    B = lambda a, b: math.exp(math.lgamma(a) + math.lgamma(b) - math.lgamma(a + b))
    return math.exp(sum(j * math.log(2 ** j * B((j + 1) / 2, (j + 1) / 2)) for j in range(1, k)))


for arg in sys.argv[1:]:
    f = arg.split(":")
    k = int(f[0]); seeds = int(f[1]) if len(f) > 1 else 3
    N = int(f[2]) if len(f) > 2 else 4096; eps = float(f[3]) if len(f) > 3 else 0.1
    S = sw.Spectrahedron.from_instance(specgen.elliptope(k))
    for s in range(seeds):
        t0 = time.time()
        r = S.volume(eps, s, N)
        print(json.dumps(dict(k=k, n=k * (k - 1) // 2, seed=s, chains=N, eps=eps, volume=r["volume"],
                              closed=closed(k), ratio=r["volume"] / closed(k), std_rel=r["std_rel"],
                              phases=r["phases"], calls=r["calls"], seconds=time.time() - t0)), flush=True)
