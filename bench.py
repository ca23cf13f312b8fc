#!/usr/bin/env python3
"""Benchmark of the B200 HPS leaf stage (arXiv 2211.14969, BASELINE.json metric).

One "step" = batched static condensation of every leaf of the workload's mesh
(K1 assembly + K2/K3 fused LU/TRSM/Schur), i.e. the reference's
batched_condense.  Default workload: config C4 (p=42, 98x98
leaves, kappa=500, crystal b(x), ~16.2M DOF) -- the configuration the
north-star target (>=60% FP64 peak, leaf-sharded 1/2/4/8 GPUs) is stated on.
`--config C2` runs p=22 (configs[1]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

N>1: launched with torchrun, one rank per GPU; leaves are sharded by contiguous
element range (strong scaling, no collective on the data path); timing is the
max over ranks of CUDA-event time on the launching stream.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2211_14969_b200 import problems as P  # noqa: E402

METRIC = "leaf-condensation leaves/s & DOF/s at p=22/42 (1/2/4/8 B200), FP64 TFLOP/s vs peak"
def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6552.0   # B200 measured copy bandwidth (MEASURED_PEAKS.json of this pool)


hbm_peak = _hbm_peak()
FP64_PEAK_TFLOPS = 37.1   # fallback: DMMA m8n8k4 loop on this pool's B200 (profiles/r01_fp64_peak.log)
FP64_PEAK_NOTE = ("measured in this run on this GPU: register-only DMMA m8n8k4 loop run back to back for 3 s "
                  "(sustained, hps_gpu_fp64_peak_tflops_sustained; K2 is timed inside a long step), burst figure "
                  "beside it (MEASURED_PEAKS.json and B200_PROFILING.md have no FP64 figure)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--leaf-solve", action=argparse.BooleanOptionalAction, default=True,
                    help="also time batched leaf_solve (K5, recompute policy) on the workload")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def shard(n, world, rank):
    base, rem = divmod(n, world)
    e0 = rank * base + min(rank, rem)
    return e0, e0 + base + (1 if rank < rem else 0)


def leaf_inputs(cfg, e0, e1):
    """Synthetic b = crystal field, f = 0 (SURVEY §8d timing inputs)."""
    X, Y = P.leaf_coords(cfg["nx"], cfg["ny"], cfg["p"], cfg["a"], elements=np.arange(e0, e1))
    if cfg["kappa"] == 0.0:
        b = np.ones_like(X)
    else:
        b = P.crystal_field(X, Y)
    f = np.zeros_like(X)
    return np.ascontiguousarray(b), np.ascontiguousarray(f)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def gpu_index(local_rank):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids):
            return ids[local_rank]
    return str(local_rank)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def b_star(cfg):
    """Resonant coefficient value of the workload: kappa^2 b* = lowest interior Dirichlet
    eigenvalue of a leaf of side a, ~2 pi^2 / a^2 (189,575 at C4 vs 2 pi^2 98^2 = 189,571)."""
    if cfg["kappa"] == 0.0:
        return float("inf")   # Laplace: no interior resonance
    return 2.0 * np.pi ** 2 / (cfg["a"] ** 2 * cfg["kappa"] ** 2)


def sample_order(cfg, b):
    """Leaves for the CPU sample, most demanding first: those whose b range spans the resonant
    b*, then the rest of the crystal (b not identically 1), then the b = 1 leaves; each group
    in a fixed pseudo-random order."""
    rng = np.random.default_rng(7)
    bmin, bmax = b.min(axis=1), b.max(axis=1)
    bs = b_star(cfg)
    near = (bmin <= bs) & (bmax >= bs)
    var = (bmin < 1.0) & ~near
    rest = ~(near | var)
    groups = [rng.permutation(np.nonzero(m)[0]) for m in (near, var, rest)]
    return np.concatenate(groups), int(near.sum()), int((bmin < 1.0).sum())


def cpu_baseline(cfg, seconds, b_all, T_dev=None, threads=0):
    """The CPU oracle (C++ restatement of SPEC batched_condense, OpenBLAS, all host threads via
    the reference's parallel_for contract) on a bounded sample of the same workload: the
    sample starts with the near-resonant and crystal leaves (sample_order).  When the device
    arm's T (all leaves of this rank, f = 0 so w = 0) is given, the sample doubles as a parity
    check of the GPU output against the oracle (relative Frobenius per leaf, bar 1e-10).
    Returns (leaves/s, cores, sample description, parity dict or None)."""
    from oracle import pyoracle as O
    cores = threads or O.hardware_workers()
    p = cfg["p"]
    order, n_near, n_var = sample_order(cfg, b_all)
    batch = max(cores, 1)
    done, t_total = 0, 0.0
    errs, status_mismatch, minratio = [], 0, np.inf
    f0 = np.zeros((batch, p * p))
    while done < order.size and (t_total < seconds or done < 2 * batch):
        ids = order[done:done + batch]
        bb = np.ascontiguousarray(b_all[ids])
        t0 = time.perf_counter()
        r = O.batched_condense(p, cfg["a"], cfg["kappa"], bb, f0[:ids.size], workers=cores,
                               raise_on_resonance=False)
        t_total += time.perf_counter() - t0
        done += ids.size
        minratio = min(minratio, float(r["min_pivot_ratio"].min()))
        if T_dev is not None:
            Tg = T_dev[ids].reshape(ids.size, -1)
            Tr = r["T"].reshape(ids.size, -1)
            ok = r["status"] == 0
            num = np.linalg.norm(Tg - Tr, axis=1)
            den = np.maximum(np.linalg.norm(Tr, axis=1), 1e-300)
            errs.extend((num / den)[ok].tolist())
    sample = (f"{done} of {cfg['n_leaves']} leaves of {cfg['name']} (p={p}): the {min(done, n_near)} leaves "
              f"whose b spans b*={b_star(cfg):.4g}, then crystal leaves ({n_var} with b != 1 in the mesh), "
              f"{t_total:.1f} s wall")
    parity = None
    if T_dev is not None and errs:
        parity = {"leaves": len(errs), "near_resonant_in_sample": int(min(done, n_near)),
                  "max_relfro_T": max(errs), "median_relfro_T": float(np.median(errs)),
                  "min_pivot_ratio": minratio, "bar": 1e-10, "pass": max(errs) <= 1e-10,
                  "inputs": "device arm's T (crystal b, f=0) vs oracle on the CPU sample"}
    return done / t_total, cores, sample, parity


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import pyoracle as O
    cores = O.hardware_workers()
    p = cfg["p"]
    # bounded sample per step (~4 s of all-core work) from the same leaf order as the
    # cpu_baseline leg: near-resonant leaves, then the crystal, then b = 1 leaves
    b_all, _ = leaf_inputs(cfg, 0, cfg["n_leaves"])
    order, _, _ = sample_order(cfg, b_all)
    f = np.zeros((cores, p * p))
    t0 = time.perf_counter()
    O.batched_condense(p, cfg["a"], cfg["kappa"], b_all[order[:cores]], f, workers=cores,
                       raise_on_resonance=False)
    per_round = time.perf_counter() - t0
    rounds = max(1, int(4.0 / max(per_round, 1e-3)))
    n = min(cfg["n_leaves"], rounds * cores)
    b = np.ascontiguousarray(b_all[order[:n]])
    f = np.zeros_like(b)
    del b_all
    for _ in range(args.warmup):
        O.batched_condense(p, cfg["a"], cfg["kappa"], b, f, workers=cores, raise_on_resonance=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.batched_condense(p, cfg["a"], cfg["kappa"], b, f, workers=cores, raise_on_resonance=False)
    dt = (time.perf_counter() - t0) / args.steps
    v = n / dt
    sample = (f"{n} of {cfg['n_leaves']} leaves of {cfg['name']} per step (near-resonant and crystal "
              f"leaves first); host CPU: {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "leaves/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, args.gpus),
        "dof_per_s": v * cfg["N"] / cfg["n_leaves"],
        "tflops": v * P.flops_condense(p) / 1e12,
        "cpu_baseline": {"value": v, "unit": "leaves/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "leaves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference has no implementation (SPEC + headers only); the arm times the C++ restatement "
                "of SPEC batched_condense (oracle/, OpenBLAS, parallel_for over all host threads)",
    }
    print(json.dumps(line), flush=True)


def k2_kernel_name(p):
    """The condensation kernel the C-ABI dispatches for p (hps_kernels.h small_condense_preferred)."""
    if 4 <= p <= 12:
        return "k2s_condense_kernel (register-resident, fused assembly, DFMA f64)"
    if (p - 2) ** 2 + 4 * (p - 1) <= 640:
        return "g128::k2_lu_lockstep_kernel (4 leaves per CTA, DMMA f64)"
    return "g256::k2_lu_schur_kernel (DMMA f64)"


def workload_config(cfg, n_gpus):
    return {"workload": f"{cfg['name']}: batched_condense p={cfg['p']}, {cfg['nx']}x{cfg['ny']} leaves, "
                        f"kappa={cfg['kappa']}, crystal b(x), f=0",
            "p": cfg["p"], "nx": cfg["nx"], "ny": cfg["ny"], "kappa": cfg["kappa"], "leaves": cfg["n_leaves"],
            "dof": cfg["N"], "parallelism": f"leaf-range shard x{n_gpus}",
            "l2": l2_note(cfg)}


def l2_note(cfg):
    """Each step streams every leaf's augmented operator (K1 writes it, K2 factors it in place):
    the per-step HBM working set is leaves x workspace bytes, far above the 126 MB L2."""
    p = cfg["p"]
    ni, nb = (p - 2) ** 2, 4 * (p - 1)
    nblk = (ni + 63) // 64
    ld = ((64 * nblk + nb + 1) + 63) // 64 * 64
    rpad = ((ni + nb) + 63) // 64 * 64
    ws = rpad * ld * 8
    return (f"inputs larger than L2: per-step workspace {ws / 1e6:.2f} MB/leaf x {cfg['n_leaves']} leaves "
            f"= {ws * cfg['n_leaves'] / 1e9:.1f} GB streamed per step (no flush needed)")


def main():
    args = parse()
    cfg = P.config(args.config)
    cfg["name"] = args.config
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import torch.distributed as dist
    from paper_2211_14969_b200 import leaf_gpu as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    p = cfg["p"]
    e0, e1 = shard(cfg["n_leaves"], world, rank)
    n = e1 - e0
    nb = 4 * (p - 1)
    b, f = leaf_inputs(cfg, e0, e1)
    stage = G.LeafStage(p, cfg["nx"], cfg["ny"], cfg["kappa"], a=cfg["a"], device=local)
    info = stage.info()
    try:
        peak_burst = G.fp64_peak_tflops(local)
        peak = G.fp64_peak_tflops(local, sustained_s=3.0)
        peak_note = FP64_PEAK_NOTE
    except Exception:
        peak_burst = None
        peak, peak_note = FP64_PEAK_TFLOPS, "fallback: profiles/r01_fp64_peak.log (live probe failed)"

    # ---- device-resident arm (value) ----
    dev = torch.device("cuda", local)
    d_b = torch.from_numpy(b).to(dev)
    d_f = torch.from_numpy(f).to(dev)
    d_T = torch.empty((n, nb, nb), dtype=torch.float64, device=dev)
    d_w = torch.empty((n, nb), dtype=torch.float64, device=dev)
    d_s = torch.empty((n,), dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)  # non-default stream: the C-ABI launches on it

    def step():
        stage.condense_device(e0, n, d_b.data_ptr(), d_f.data_ptr(), d_T.data_ptr(), d_w.data_ptr(),
                              d_s.data_ptr(), stream.cuda_stream)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    bad = int((d_s != 0).sum().item())
    clocks = ClockSampler(gpu_index(local))
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    stage.reset_timing()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    tim = stage.timing()
    ms_max = max_over_ranks(ms)
    k2_ms = tim["ms_lu_schur"] / args.steps
    kernels = tim["kernels"]

    # ---- end-to-end arm (host buffers through the public C-ABI) ----
    e2e = None
    if not args.no_e2e:
        pb = G.PinnedArray(b.shape); pb.array[:] = b
        pf = G.PinnedArray(f.shape); pf.array[:] = f
        pT = G.PinnedArray((n, nb, nb)); pw = G.PinnedArray((n, nb))
        for _ in range(max(1, min(args.warmup, 2))):
            stage.condense(pb.array, pf.array, e0=e0, out=(pT.array, pw.array), raise_on_resonance=False)
        k_e2e = args.steps
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            stage.condense(pb.array, pf.array, e0=e0, out=(pT.array, pw.array), raise_on_resonance=False)
        dt = time.perf_counter() - t0
        barrier()
        dt_max = max_over_ranks(dt)
        e2e = {"value": cfg["n_leaves"] * k_e2e / dt_max, "unit": "leaves/s",
               "h2d_bytes_per_step": int(2 * cfg["n_leaves"] * p * p * 8),
               "d2h_bytes_per_step": int(cfg["n_leaves"] * (nb * nb + nb) * 8 + 4 * cfg["n_leaves"]),
               "steps": k_e2e, "api": "hps_gpu_condense (pinned host b,f -> T,w)"}
        for a in (pb, pf, pT, pw):
            a.free()

    # ---- K5: batched leaf_solve (recompute policy) through the C-ABI ----
    leaf_solve = None
    if args.leaf_solve:
        rng = np.random.default_rng(3)
        v = rng.uniform(-1.0, 1.0, (n, nb))
        pb = G.PinnedArray(b.shape); pb.array[:] = b
        pf = G.PinnedArray(f.shape); pf.array[:] = f
        pv = G.PinnedArray(v.shape); pv.array[:] = v
        pu = G.PinnedArray((n, p * p))
        stage.leaf_solve(pb.array, pf.array, pv.array, e0=e0, out=pu.array)   # warm-up
        k_ls = max(1, min(args.steps, 3))
        dev_ms, k1_ms, k2k5_ms = 0.0, 0.0, 0.0
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_ls):
            stage.leaf_solve(pb.array, pf.array, pv.array, e0=e0, out=pu.array)
            tl = stage.timing()
            dev_ms += tl["ms_total"]; k1_ms += tl["ms_assemble"]; k2k5_ms += tl["ms_lu_schur"]
        dt = max_over_ranks(time.perf_counter() - t0)
        ni = (p - 2) ** 2
        f_ls = P.flops_leaf_solve(p)
        leaf_solve = {"api": "hps_gpu_leaf_solve (recompute: K1s assemble [A_ii | f - A_ib v], K2 LU + forward "
                             "solve, K5 back substitution; pinned host b, f, v -> u)",
                      "steps": k_ls, "e2e_leaves_per_s": cfg["n_leaves"] * k_ls / dt,
                      "device_leaves_per_s": n * k_ls / (dev_ms / 1e3),
                      "ms_per_step_device": dev_ms / k_ls, "ms_assemble": k1_ms / k_ls,
                      "ms_lu_backsolve": k2k5_ms / k_ls,
                      "roofline": {"bound": "tensor", "flops_per_leaf": f_ls,
                                   "achieved": n * f_ls / (k2k5_ms / k_ls / 1e3) / 1e12, "peak": peak,
                                   "unit": "TFLOP/s",
                                   "frac": n * f_ls / (k2k5_ms / k_ls / 1e3) / 1e12 / peak,
                                   "note": "F_leafsolve = 2/3 n_i^3 + 2 n_i^2 + 2 n_i n_b (SURVEY 8d) over the "
                                           "K2+K5 device time"},
                      "h2d_bytes_per_step": int(n * (2 * p * p + nb) * 8), "d2h_bytes_per_step": int(n * p * p * 8)}
        for a_ in (pb, pf, pv, pu):
            a_.free()

    # ---- secondary: C2 (p=22, configs[1]) device-resident, same K/W ----
    secondary = None
    if args.config == "C4":
        c2 = P.config("C2"); c2["name"] = "C2"
        s0, s1 = shard(c2["n_leaves"], world, rank)
        b2, f2 = leaf_inputs(c2, s0, s1)
        st2 = G.LeafStage(22, c2["nx"], c2["ny"], c2["kappa"], a=c2["a"], device=local)
        nb2 = 84
        db2 = torch.from_numpy(b2).to(dev); df2 = torch.from_numpy(f2).to(dev)
        dT2 = torch.empty((s1 - s0, nb2, nb2), dtype=torch.float64, device=dev)
        dw2 = torch.empty((s1 - s0, nb2), dtype=torch.float64, device=dev)
        ds2 = torch.empty((s1 - s0,), dtype=torch.int32, device=dev)

        def step2():
            st2.condense_device(s0, s1 - s0, db2.data_ptr(), df2.data_ptr(), dT2.data_ptr(), dw2.data_ptr(),
                                ds2.data_ptr(), stream.cuda_stream)
        for _ in range(args.warmup):
            step2()
        barrier(); torch.cuda.synchronize()
        st2.reset_timing()
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            step2()
        a1.record(stream)
        torch.cuda.synchronize(); barrier()
        ms2 = max_over_ranks(a0.elapsed_time(a1))
        t2 = st2.timing()
        v2 = c2["n_leaves"] * args.steps / (ms2 / 1e3)
        secondary = {"config": "C2: p=22, 48x48 leaves, kappa=100", "value": v2, "unit": "leaves/s",
                     "dof_per_s": v2 * c2["N"] / c2["n_leaves"],
                     "tflops": v2 * P.flops_condense(22) / 1e12,
                     "k2_tflops": (s1 - s0) * P.flops_condense(22) / (t2["ms_lu_schur"] / args.steps / 1e3) / 1e12,
                     "k2_frac": (s1 - s0) * P.flops_condense(22) / (t2["ms_lu_schur"] / args.steps / 1e3) / 1e12 / peak,
                     "ms_per_step": ms2 / args.steps}
        st2.close()

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu, parity = None, None
    if world == 1 and not args.no_cpu:
        v, cores, sample, parity = cpu_baseline(cfg, args.cpu_seconds, b, T_dev=d_T.cpu().numpy())
        cpu = {"value": v, "unit": "leaves/s", "cores": cores, "kind": "port", "sample": sample,
               "cpu_model": cpu_model()}

    # ---- storage policy 's_solve' (PAPER.md:162-165 trade study): condense also keeps
    # [S_solve | A_ii^-1 f] per leaf (K3), leaf_solve is one HBM-bound GEMV per leaf (K5s) ----
    stored = None
    if args.leaf_solve:
        stage.close()
        torch.cuda.empty_cache()
        try:
            st3 = G.LeafStage(p, cfg["nx"], cfg["ny"], cfg["kappa"], a=cfg["a"], device=local,
                              storage=G.STORAGE_S_SOLVE)
            n3 = n
            pb = G.PinnedArray(b.shape); pb.array[:] = b
            pf = G.PinnedArray(f.shape); pf.array[:] = f
            pT = G.PinnedArray((n3, nb, nb)); pw = G.PinnedArray((n3, nb))
            v3 = np.random.default_rng(3).uniform(-1.0, 1.0, (n3, nb))
            pv = G.PinnedArray(v3.shape); pv.array[:] = v3
            pu = G.PinnedArray((n3, p * p))
            st3.condense(pb.array, pf.array, e0=e0, out=(pT.array, pw.array), raise_on_resonance=False)
            t3 = st3.timing()
            st3.leaf_solve(pb.array, pf.array, pv.array, e0=e0, out=pu.array)   # warm-up
            ks = 5
            dev_ms = 0.0
            t0 = time.perf_counter()
            for _ in range(ks):
                st3.leaf_solve(pb.array, pf.array, pv.array, e0=e0, out=pu.array)
                dev_ms += st3.timing()["ms_lu_schur"]
            dt = time.perf_counter() - t0
            ni = (p - 2) ** 2
            byts = 8 * (ni * (nb + 1) + nb + p * p)
            stored = {"policy": "s_solve (HPS_STORAGE_S_SOLVE)",
                      "condense_device_ms": t3["ms_total"],
                      "condense_leaves_per_s_device": n3 / (t3["ms_total"] / 1e3),
                      "store_bytes": int(n3 * ni * (nb + 1) * 8),
                      "leaf_solve_e2e_leaves_per_s": n3 * ks / dt,
                      "leaf_solve_device_ms": dev_ms / ks,
                      "leaf_solve_device_leaves_per_s": n3 / (dev_ms / ks / 1e3),
                      "k5s_roofline": {"bound": "hbm", "bytes_per_leaf": byts,
                                       "achieved": n3 * byts / (dev_ms / ks / 1e3) / 1e9,
                                       "peak": hbm_peak, "unit": "GB/s",
                                       "frac": n3 * byts / (dev_ms / ks / 1e3) / 1e9 / hbm_peak}}
            for a_ in (pb, pf, pT, pw, pv, pu):
                a_.free()
            st3.close()
        except Exception as ex:   # e.g. the store does not fit next to the workspace
            stored = {"policy": "s_solve", "skipped": str(ex)[:200]}

    if rank == 0:
        value = cfg["n_leaves"] * args.steps / (ms_max / 1e3)
        f_leaf = P.flops_condense(p)
        achieved = n * f_leaf / (k2_ms / 1e3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", f"k2_traffic_p{p}.json")
        if os.path.exists(tpath):
            try:   # ncu dram bytes per leaf x leaves of the average K2 launch (chunk)
                chunks = max(1, -(-n // info["chunk_leaves"]))
                traffic = json.load(open(tpath))["bytes_per_leaf"] * n / chunks
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": "leaves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world),
            "dof_per_s": value * cfg["N"] / cfg["n_leaves"],
            "tflops": value * f_leaf / 1e12,
            "fp64_peak_frac": value * f_leaf / 1e12 / (peak * world),
            "roofline": {"bound": "tensor", "kernel": k2_kernel_name(p), "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_note, "peak_burst": peak_burst,
                         "flops_per_leaf": f_leaf, "k2_ms_per_step_rank0": k2_ms,
                         "traffic_unit": "DRAM bytes per K2 launch (ncu, scaled to the launch's leaves)",
                         "k1_ms_per_step_rank0": tim["ms_assemble"] / args.steps},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": kernels,
            "clocks": clk,
            "resonant_leaves_rank0": bad,
            "chunk_leaves": info["chunk_leaves"],
            "secondary": secondary,
            "leaf_solve": leaf_solve,
            "leaf_solve_stored_s_solve": stored,
        }
        print(json.dumps(line), flush=True)
    stage.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
