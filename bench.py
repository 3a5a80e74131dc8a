"""bench.py -- boundary-oracle calls/s of the billiard walk at n = m = 100
(BASELINE.json metric, first half) on the M100 workload, through the C-ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one scheduler round over the whole chain population: every chain
makes exactly one boundary-oracle call (K1 A(v) GEMM -> K2 chord/advance ->
K3 normal GEMM -> K4 reflect), i.e. one pass of the hot path over the batch.
All 65536 chains stay active for the whole timed region (a chain needs ~27000
rounds to finish its 100 steps), so every timed round processes the full batch.

N > 1 (torchrun): the 65536 chains of the workload are split into N contiguous
global-id ranges (configs[4]: "65536 chains ... sharded across 1/2/4/8 B200"),
rank r runs [r*65536/N, (r+1)*65536/N) (the ids key the RNG, so a chain's
trajectory does not depend on N), no collective in the data path:
"scaling": "strong" (total work fixed).  --scaling weak runs 65536 chains per rank.
Timing: barrier + cuda synchronize on both sides, CUDA events on the library
stream, max over ranks.

--impl reference times the CPU oracle (oracle/, plain C, Jacobi) on the host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DIM = M_DIM = 100
CHAINS = 65536
STEPS_PER_CHAIN = 100
SEED = 4
INSTANCE_SEED = 3  # BASELINE.json configs[3] instance (SURVEY 8(d).1 "M100")
L_TAU = 2.0 * math.sqrt(N_DIM)
RHO = 10 * N_DIM
HMC_L = 1.09  # configs[3] HMC trajectory length: the diameter estimate
CHMC_L, CHMC_Q, CHMC_H = 2.0, 3, 0.25  # collocation HMC-r side line (R33)
LANCZOS_K = 55  # SURVEY V9 prior; the bench uses the device-measured mean J of its timed rounds

WORKLOAD = (f"M100: billiard walk (Alg. 5) on the BASELINE.json configs[3] instance (rand-cube n=m={N_DIM}, "
            f"seed {INSTANCE_SEED}), {CHAINS} chains x {STEPS_PER_CHAIN} steps, L=2sqrt(n), rho=10n, seed {SEED}")


def flops_per_call(n: int, m: int, k: int = LANCZOS_K) -> dict:
    """SURVEY 8(d).2 algorithmic flops of one line boundary-oracle call that reflects."""
    contr = 2 * n * m * (m + 1)  # A(v) and normal contractions (packed symmetric)
    k2 = m ** 3 / 3 + m ** 3 + 2 * k * m * m  # Cholesky + congruence + Lanczos matvecs
    return dict(total=contr + k2, k2=k2, k1=n * m * (m + 1), k3=n * m * (m + 1), lanczos=2 * k * m * m)


def ncu_traffic_per_launch(tag: str, kernel: str = ""):
    """DRAM bytes (read + write) of one launch of the dominant kernel, from the latest
    committed ncu --set full summary profiles/*<tag>.txt (tools/summarize_ncu.py), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*{tag}*.txt")))
    if not files:
        return None
    vals = {}
    units = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    cur = ""
    for line in open(files[-1]):
        if line.startswith("# kernel:"):
            cur = line
            continue
        if kernel and cur and kernel not in cur:
            continue
        parts = [p.strip() for p in line.split("|")]
        if len(parts) == 4 and parts[0] == "raw" and parts[1] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                vals[parts[1]] = float(parts[3].replace(",", "")) * units.get(parts[2], 1.0)
            except ValueError:
                pass
    if len(vals) != 2:
        return None
    return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"], "unit": "B/launch",
            "source": os.path.relpath(files[-1], ROOT)}


def measured_fp64() -> dict:
    """The committed FP64 measurements of this pool's B200 (tools/fp64_peak.py on the box:
    cuBLAS DGEMM 8192^3 burst / 4-s sustained, DFMA and DMMA issue loops)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*fp64_peak.json")))
    if not files:
        return {}
    d = json.load(open(files[-1]))
    d["source"] = os.path.relpath(files[-1], ROOT)
    return d


def fp64_peak_tflops() -> float:
    """FP64 FMA pipe peak derived from unit counts and clocks (B200: 148 SMs x 64
    DFMA/clk x 2 flop x 1.965 GHz).  MEASURED_PEAKS.json carries
    no fp64 entry; the measured DGEMM / DMMA rates are reported beside it."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        mhz = float(mp.get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_sample(seconds: float = 15.0, nthreads: int = 0) -> dict:
    """Oracle (plain C, Jacobi) boundary-oracle calls/s on the M100 instance, on
    the host cores: each thread runs the billiard walk of one chain (same seed
    and chain ids as the GPU run) and counts oracle calls until the budget ends
    (bounded by the trace length)."""
    import oracle
    import specgen
    from concurrent.futures import ThreadPoolExecutor

    nthreads = nthreads or (os.cpu_count() or 1)
    inst = specgen.config_instance(3)
    lmi = oracle.Lmi(inst)
    # calibrate: one call
    t0 = time.time()
    oracle.chord(lmi, np.zeros(N_DIM), specgen.unit_vectors(1, N_DIM, 0)[0])
    per_call = max(time.time() - t0, 1e-3)
    max_refl = max(2, int(seconds / per_call / 1.2))

    def one(c):
        tr = oracle.trace(lmi, oracle.BILLIARD, SEED, c, 1000, L_TAU, RHO, max_refl)
        return tr["calls"]  # every oracle call made (the walk completes the last step)

    t0 = time.time()
    with ThreadPoolExecutor(nthreads) as ex:
        recs = list(ex.map(one, range(nthreads)))
    wall = time.time() - t0
    calls = int(sum(recs))
    return {"value": calls / wall, "unit": "calls/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{nthreads} chains x the steps holding their first {max_refl} reflections of the M100 walk "
                      f"(seed {SEED}), {calls} oracle calls in {wall:.1f} s"}


def run_reference(args):
    """The oracle (plain C, Jacobi) as it stands, on the host cores: each step runs one M100
    billiard chain per core (global chain ids step*cores + t, seed 4) for a bounded number of
    boundary-oracle calls (the first REF_CALLS reflections), so that --steps K --warmup W
    finishes in minutes.  Rank 0 only under torchrun."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    import specgen
    from concurrent.futures import ThreadPoolExecutor

    nthreads = os.cpu_count() or 1
    inst = specgen.config_instance(3)
    lmi = oracle.Lmi(inst)
    ref_calls = int(os.environ.get("SPECWALK_REF_CALLS", "16"))

    def one(chain):
        # exactly ref_calls boundary-oracle calls of chain `chain` of the M100 walk (oracle.replay)
        _, calls = oracle.replay(lmi, oracle.BILLIARD, SEED, chain, STEPS_PER_CHAIN, L_TAU, RHO, ref_calls)
        return calls

    ex = ThreadPoolExecutor(nthreads)
    for s in range(args.warmup):
        list(ex.map(one, range(s * nthreads, (s + 1) * nthreads)))
    t0 = time.time()
    total = 0
    for s in range(args.steps):
        base = (args.warmup + s) * nthreads
        total += sum(ex.map(one, range(base, base + nthreads)))
    wall = time.time() - t0
    value = total / wall
    line = {
        "impl": "reference", "metric": "boundary-oracle calls/s (billiard walk, n=m=100)", "value": value,
        "unit": "calls/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall * 1e3 / max(args.steps, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": N_DIM, "m": M_DIM,
                   "reference_step": f"{nthreads} M100 billiard chains (one per host core), the first {ref_calls} "
                                     f"boundary-oracle calls of each (oracle/: plain C, Jacobi)"},
        "cpu_baseline": {"value": value, "unit": "calls/s", "cores": nthreads, "kind": "oracle",
                         "sample": f"{args.steps} steps x {nthreads} chains x {ref_calls} calls = {total} calls"},
        "e2e": {"value": value, "unit": "calls/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch

    world, rank, local = _dist()
    if world > 1:
        import torch.distributed as dist
        # SPECWALK_DIST_TEST=1: logic test of the N > 1 path on a 1-GPU box (every rank on
        # cuda:0, gloo collectives; ranks are independent until the final reductions)
        test1 = os.environ.get("SPECWALK_DIST_TEST") == "1"
        if test1:
            local = 0
        torch.cuda.set_device(local)
        if test1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        coll_dev = "cpu" if test1 else "cuda"
    else:
        dist = None
        coll_dev = "cuda"
        torch.cuda.set_device(0)
    import paper_2010_03817_b200 as sw
    import specgen

    dev = torch.cuda.current_device()
    inst = specgen.config_instance(3)
    S = sw.Spectrahedron.from_instance(inst, device=dev)
    strong = (args.scaling == "strong")
    if strong:
        if args.chains % world:
            raise SystemExit(f"--chains {args.chains} does not split over {world} ranks")
        local_chains = args.chains // world
    else:
        local_chains = args.chains
    begin = rank * local_chains
    chains = local_chains * world
    stream = torch.cuda.ExternalStream(S.stream(), device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident run: warm-up rounds, then K timed rounds
    S.walk_begin(local_chains, STEPS_PER_CHAIN, L_TAU, RHO, SEED, chain_begin=begin)
    S.walk_rounds(max(args.warmup, 3) if args.warmup > 0 else 0)
    st0 = S.walk_stats_now()
    S.kernel_timing(True)
    S.lanczos_iterations(reset=True)
    launches0 = S.kernel_launches()
    barrier()
    with ClockSampler(dev) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        active = S.walk_rounds(args.steps)
        e1.record(stream)
        e1.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = S.kernel_launches() - launches0
    st1 = S.walk_stats_now()
    lz = S.lanczos_iterations(reset=True)
    kt = S.kernel_times()
    S.kernel_timing(False)
    S.walk_end()
    calls = st1["calls"] - st0["calls"]
    t = torch.tensor([ms, float(calls)], dtype=torch.float64, device=coll_dev)
    if dist is not None:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms_max, calls_tot = float(tmax[0]), float(t[1])
    else:
        ms_max, calls_tot = ms, float(calls)
    value = calls_tot / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel, from its own events on the library stream:
    # K2b lanczos_kernel when K2 is split (m = 100), else the whole K2
    J = lz["mean_j"] if lz["solves"] > 0 else float(LANCZOS_K)  # measured k of the flop model
    f = flops_per_call(N_DIM, M_DIM, J)
    k2_ms = kt["ms"]["K2_chord"]
    k2_launches = kt["launches"]["K2_chord"]
    k2_items = kt["k2_items"]
    k2_avg_ms = k2_ms / max(k2_launches, 1)
    items_per_launch = k2_items / max(k2_launches, 1)
    k2_flops_per_launch = f["k2"] * items_per_launch
    k2_achieved = k2_flops_per_launch / (k2_avg_ms * 1e-3) / 1e12
    peak = fp64_peak_tflops()
    meas = measured_fp64()
    phases = kt.get("k2_phases_ms", {})
    share = {k: v / max(sum(kt["ms"].values()), 1e-9) for k, v in kt["ms"].items()}
    tot_ms = max(sum(kt["ms"].values()), 1e-9)
    for k, v in phases.items():
        share[k] = v / tot_ms
    k2cfg = S.k2_config()
    if phases.get("K2b_lanczos", 0.0) > 0.0:
        dom = "K2b " + ("lanczos2_kernel (256 threads, 2 CTAs/SM)" if "lanczos2" in k2cfg else "lanczos_kernel<512,13>")
        dom_ms = phases["K2b_lanczos"]
        dom_flops = f["lanczos"]
    else:
        dom, dom_ms, dom_flops = "K2 chord_kernel2 (fused)", k2_ms, f["k2"]
    dom_avg_ms = dom_ms / max(k2_launches, 1)
    achieved = dom_flops * items_per_launch / (dom_avg_ms * 1e-3) / 1e12
    tr = ((ncu_traffic_per_launch("lanczos2_full_ncu", "lanczos2_kernel") if "lanczos2" in dom
           else ncu_traffic_per_launch("lanczos_full_ncu", "lanczos_kernel")) if dom.startswith("K2b") else None)
    traffic = tr["bytes"] if tr else None

    # ---- end-to-end through the public host API (walk_sample with host buffers)
    e2e = None
    if args.e2e_chains > 0:
        ec = args.e2e_chains // world if strong else args.e2e_chains
        eb = rank * ec
        x0 = np.zeros((ec, N_DIM))
        barrier()
        te0 = torch.cuda.Event(enable_timing=True)
        te1 = torch.cuda.Event(enable_timing=True)
        te0.record(stream)
        out = S.walk_sample(ec, 1, L_TAU, RHO, SEED, x0=x0, chain_begin=eb)
        te1.record(stream)
        te1.synchronize()
        barrier()
        ems = te0.elapsed_time(te1)
        et = torch.tensor([ems, float(out["stats"]["calls"])], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            emax = et.clone()
            dist.all_reduce(emax[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(et[1:], op=dist.ReduceOp.SUM)
            ems, ecalls = float(emax[0]), float(et[1])
        else:
            ecalls = float(et[1])
        e2e = {"value": ecalls / (ems * 1e-3), "unit": "calls/s", "h2d_bytes_per_step": int(x0.nbytes),
               "d2h_bytes_per_step": int(out["final_x"].nbytes + out["sum_x"].nbytes + out["sum_xx"].nbytes),
               "workload": f"walk_sample(host buffers): {args.e2e_chains} chains x 1 billiard step from x0=0 on "
                           f"the M100 instance (H2D x0, D2H end points + moments inside the region; includes the "
                           f"reflection-count tail of the step)"}

    # ---- configs[3]'s own workload (reflective HMC, T = 1, c ~ N(0, I) normalised) on the same
    # instance: HMC-r boundary-oracle calls/s over scheduler rounds (K5 split kernels)
    hmc = None
    if args.hmc_rounds > 0:
        c3 = specgen.objective(N_DIM, 3)
        S.set_objective(c3)
        S.walk_begin(local_chains, 200, HMC_L, RHO, 3, kind=sw.HMC, T=1.0, chain_begin=begin)
        S.walk_rounds(2)
        h0 = S.walk_stats_now()
        hl0 = S.kernel_launches()
        S.lanczos_iterations(reset=True)
        barrier()
        he0 = torch.cuda.Event(enable_timing=True)
        he1 = torch.cuda.Event(enable_timing=True)
        he0.record(stream)
        S.walk_rounds(args.hmc_rounds)
        he1.record(stream)
        he1.synchronize()
        barrier()
        hms = he0.elapsed_time(he1)
        h1 = S.walk_stats_now()
        hlz = S.lanczos_iterations(reset=True)
        S.walk_end()
        ht = torch.tensor([hms, float(h1["calls"] - h0["calls"])], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            hmax = ht.clone()
            dist.all_reduce(hmax[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(ht[1:], op=dist.ReduceOp.SUM)
            hms, hcalls = float(hmax[0]), float(ht[1])
        else:
            hcalls = float(ht[1])
        hcalls_local = float(h1["calls"] - h0["calls"])
        iw = hlz["solves"] / max(hcalls_local, 1.0)  # Weyl iterations per call (one N_1 Lanczos solve each)
        hJ = hlz["mean_j"]
        m_ = M_DIM
        hmc_flops = 2 * N_DIM * m_ * (m_ + 1) + iw * (m_ ** 3 / 3 + 2 * m_ ** 3 + 2 * hJ * m_ * m_)
        h_ach = hmc_flops * hcalls / (hms * 1e-3) / 1e12
        hmc = {"metric": "HMC-r boundary-oracle calls/s (configs[3]: n=m=100, T=1, c~N(0,I) normalised)",
               "value": hcalls / (hms * 1e-3), "unit": "calls/s", "chains": chains, "rounds": args.hmc_rounds,
               "roofline": {"bound": "alu", "achieved": h_ach, "peak": peak, "unit": "TFLOP/s", "frac": h_ach / peak,
                            "kernel": "whole HMC-r round (K1 + K5 split kernels + K3 + K4)",
                            "flops_per_call": hmc_flops, "weyl_iterations_per_call": iw, "lanczos_j": hJ,
                            "flop_model": "SURVEY 8(d).2: 2 n m(m+1) + I_w (m^3/3 + 2 m^3 + 2 J m^2), I_w and J "
                                          "measured on the device over the timed rounds"},
               "ms": hms, "calls": hcalls, "L": HMC_L, "gpu_launches": int(S.kernel_launches() - hl0),
               "note": "one quadratic-pencil chord per chain per round (Weyl stepping, ~5 Cholesky + Lanczos "
                       "iterations per call); device events on the library stream, max over ranks"}

    # ---- north_star's second size: configs[4] (n = m = 200, 65536 billiard chains, seed 4), calls/s
    # over scheduler rounds on the m > 112 K2 variant (split: global-scratch factor phase | lanczos_t | tail),
    # with the K2 roofline fraction
    m200 = None
    if args.m200_rounds > 0:
        inst4 = specgen.config_instance(4)
        S4 = sw.Spectrahedron.from_instance(inst4, device=dev)
        stream4 = torch.cuda.ExternalStream(S4.stream(), device=dev)
        k2cfg4 = S4.k2_config()
        S4.walk_begin(local_chains, 100, 2.0 * math.sqrt(200), 2000, SEED, chain_begin=begin)
        S4.walk_rounds(2)
        g0 = S4.walk_stats_now()
        S4.kernel_timing(True)
        S4.lanczos_iterations(reset=True)
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream4)
        S4.walk_rounds(args.m200_rounds)
        f1.record(stream4)
        f1.synchronize()
        barrier()
        fms = f0.elapsed_time(f1)
        g1 = S4.walk_stats_now()
        lz4 = S4.lanczos_iterations(reset=True)
        kt4 = S4.kernel_times()
        S4.walk_end()
        del S4
        ft = torch.tensor([fms, float(g1["calls"] - g0["calls"])], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            fmax_ = ft.clone()
            dist.all_reduce(fmax_[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(ft[1:], op=dist.ReduceOp.SUM)
            fms, fcalls = float(fmax_[0]), float(ft[1])
        else:
            fcalls = float(ft[1])
        J4 = lz4["mean_j"] if lz4["solves"] > 0 else 68.0
        f4 = flops_per_call(200, 200, J4)
        k2ms4 = kt4["ms"]["K2_chord"]
        k2_ach4 = f4["k2"] * (kt4["k2_items"] / max(k2ms4 * 1e-3, 1e-12)) / 1e12
        m200 = {"metric": "boundary-oracle calls/s (billiard walk, n=m=200, configs[4])",
                "value": fcalls / (fms * 1e-3), "unit": "calls/s", "chains": chains, "rounds": args.m200_rounds,
                "ms": fms, "calls": fcalls,
                "roofline_k2": {"bound": "alu", "achieved": k2_ach4, "peak": fp64_peak_tflops(), "unit": "TFLOP/s",
                                "frac": k2_ach4 / fp64_peak_tflops(), "flops_per_chain_call": f4["k2"],
                                "lanczos_j": J4,
                                "flop_model": "SURVEY 8(d).2: m^3/3 + m^3 + 2 J m^2, J measured on the device"},
                "kernel_share": {k: v / max(sum(kt4["ms"].values()), 1e-9) for k, v in kt4["ms"].items()},
                "k2_phases_ms": kt4.get("k2_phases_ms"), "k2_config": k2cfg4}

    # ---- collocation HMC-r (sec:hmcr P:1116-1158) on the configs[2] instance (n = m = 40),
    # truncated Gaussian exp(-|x|^2 / 2), q = 3 Chebyshev nodes (degree-4 segments), h = 0.25, 65536 chains
    chmc = None
    if args.chmc_rounds > 0:
        inst2c = specgen.config_instance(2)
        Sc = sw.Spectrahedron.from_instance(inst2c, device=dev)
        streamc = torch.cuda.ExternalStream(Sc.stream(), device=dev)
        Sc.set_potential(sw.POT_GAUSS, np.zeros(inst2c.n), 1.0)
        Sc.walk_begin(local_chains, 1000, CHMC_L, 100 * inst2c.n, SEED, chain_begin=begin, kind=sw.CHMC,
                      q=CHMC_Q, h=CHMC_H)
        Sc.walk_rounds(3)
        c0s = Sc.walk_stats_now()
        Sc.lanczos_iterations(reset=True)
        Sc.chmc_counters(reset=True)
        cl0 = Sc.kernel_launches()
        barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(streamc)
        Sc.walk_rounds(args.chmc_rounds)
        q1.record(streamc)
        q1.synchronize()
        barrier()
        cms = q0.elapsed_time(q1)
        c1s = Sc.walk_stats_now()
        clz = Sc.lanczos_iterations(reset=True)
        ccn = Sc.chmc_counters(reset=True)
        claunch = int(Sc.kernel_launches() - cl0)
        Sc.walk_end()
        del Sc
        ct = torch.tensor([cms, float(c1s["calls"] - c0s["calls"])], dtype=torch.float64, device=coll_dev)
        if dist is not None:
            cmax_ = ct.clone()
            dist.all_reduce(cmax_[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(ct[1:], op=dist.ReduceOp.SUM)
            cms, ccalls = float(cmax_[0]), float(ct[1])
        else:
            ccalls = float(ct[1])
        lcalls = float(c1s["calls"] - c0s["calls"])
        nn, mm_ = inst2c.n, inst2c.m
        dq = CHMC_Q + 1
        iwc = clz["solves"] / max(lcalls, 1.0)
        cong = ccn["congruences"] / max(lcalls, 1.0)
        cflops = (2 * dq * nn * mm_ * (mm_ + 1) / 2 + iwc * (mm_ ** 3 / 3 + 2 * clz["mean_j"] * mm_ * mm_)
                  + cong * 2 * mm_ ** 3)
        c_ach = cflops * ccalls / (cms * 1e-3) / 1e12
        chmc = {"metric": "collocation HMC-r boundary-oracle calls/s (configs[2] instance n=m=40, "
                          "exp(-|x|^2/2), q=3, h=0.25)",
                "value": ccalls / (cms * 1e-3), "unit": "calls/s", "chains": chains, "rounds": args.chmc_rounds,
                "ms": cms, "calls": ccalls, "L": CHMC_L, "gpu_launches": claunch,
                "roofline": {"bound": "alu", "achieved": c_ach, "peak": peak, "unit": "TFLOP/s",
                             "frac": c_ach / peak,
                             "kernel": "whole collocation round (K7a + the d-row DMMA contraction + K7b + K3 + K4)",
                             "flops_per_call": cflops, "weyl_iterations_per_call": iwc,
                             "congruences_per_call": cong, "lanczos_j": clz["mean_j"],
                             "picard_per_segment": ccn["picard"] / max(ccn["segments"], 1),
                             "picard_unconverged": ccn["unconverged"],
                             "flop_model": "2 d n m(m+1)/2 (contraction) + I_w (m^3/3 + 2 J m^2) + C 2 m^3 "
                                           "(C = congruences K^-1 D_j K^-T), I_w, J, C device-counted"},
                "note": "one segment (degree-4 collocation polynomial, its first boundary root in (0, h']) per "
                        "chain per round; device events on the library stream, max over ranks"}

    # ---- BASELINE metric, second half: volume time at n = m = 40 (configs[2], eps 0.1, 4096 chains/phase)
    vol = None
    if args.volume_seeds > 0:
        import paper_2010_03817_b200.parallel as par
        inst2 = specgen.config_instance(2)
        S2 = sw.Spectrahedron.from_instance(inst2, device=dev)
        if dist is not None:
            par.attach(S2)
        S2.volume(0.1, 99, 512 * world, walk_len=2, burn=4)  # warm-up
        times, vols = [], []
        for sd in range(args.volume_seeds):
            barrier()
            t0 = time.time()
            r = S2.volume(0.1, sd, 4096)
            barrier()
            times.append(time.time() - t0)
            vols.append(r)
        vol = {"metric": "volume time at n=m=40 (configs[2], eps=0.1, 4096 chains/phase)", "unit": "s",
               "seconds_mean": float(np.mean(times)),
               "seconds_sd": float(np.std(times, ddof=1)) if len(times) > 1 else None,
               "seeds": list(range(args.volume_seeds)), "seconds": times,
               "volume_mean": float(np.mean([v["volume"] for v in vols])),
               "volume_sd": float(np.std([v["volume"] for v in vols], ddof=1)) if len(vols) > 1 else None,
               "volume": [v["volume"] for v in vols], "std_rel": [v["std_rel"] for v in vols],
               "phases": [v["phases"] for v in vols], "oracle_calls": [v["calls"] for v in vols],
               "paper_context": "PAPER Table 2 S-40-40: 6.7 s on an i7-6700 for the paper's own (elongated) instance"}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    cpu = cpu_oracle_sample(args.cpu_seconds) if (world == 1 and args.cpu_seconds > 0) else None
    line = {
        "metric": "boundary-oracle calls/s (billiard walk, n=m=100)",
        "value": value,
        "unit": "calls/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / max(args.steps, 1),
        "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": N_DIM, "m": M_DIM, "chains": chains, "L": L_TAU, "rho": RHO,
                   "seed": SEED, "step": "one scheduler round: one boundary-oracle call per chain",
                   "l2": "inputs larger than L2 (chain state ~10.6 GB >> 126 MB L2; no flush)",
                   "chains_per_gpu": local_chains,
                   "parallelism": f"{world} GPU(s) x {local_chains} chains, sharded by global chain id"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": dom, "k2_config": k2cfg,
                     "flops_per_chain_call": dom_flops, "chain_calls_per_launch": items_per_launch,
                     "avg_launch_ms": dom_avg_ms,
                     "lanczos_j": J,
                     "flop_model": "SURVEY 8(d).2: Lanczos 2 J m^2 for K2b; K2 total m^3/3 + m^3 + 2 J m^2; J = "
                                   "device-measured mean Lanczos iterations per solve over the timed rounds",
                     "traffic_note": ("dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                                      f"capture {tr['source'] if tr else '-'} (one 65536-chain round); algorithmic "
                                      f"bytes = M read once, {8 * M_DIM * M_DIM * items_per_launch:.3g} B/launch"),
                     "peak_note": "derived: fp64 pipe 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (MEASURED_PEAKS.json "
                                  "has no fp64 entry)",
                     "measured_fp64": meas,
                     "frac_of_measured_dgemm_sustained": (achieved / meas["dgemm_tflops_sustained"])
                     if meas.get("dgemm_tflops_sustained") else None},
        "roofline_k2_total": {"bound": "alu", "achieved": k2_achieved, "peak": peak, "unit": "TFLOP/s",
                              "frac": k2_achieved / peak, "flops_per_chain_call": f["k2"],
                              "avg_launch_ms": k2_avg_ms},
        "kernel_share": share,
        "path_tflops": value * f["total"] / 1e12,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "walk": {"calls_timed": calls_tot, "reflections": st1["reflections"], "steps_done": st1["steps"],
                 "active_chains": active},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "volume_n40": vol,
        "hmc_configs3": hmc,
        "m200_configs4": m200,
        "chmc_configs2": chmc,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chains", type=int, default=CHAINS,
                    help="global chains (strong scaling, split over ranks) or chains per GPU (weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--e2e-chains", type=int, default=65536)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--volume-seeds", type=int, default=10)
    ap.add_argument("--hmc-rounds", type=int, default=4)
    ap.add_argument("--m200-rounds", type=int, default=3)
    ap.add_argument("--chmc-rounds", type=int, default=3)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
