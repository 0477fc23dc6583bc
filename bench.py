"""bench.py -- HOOI / Multislice-Projection sweep throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = the whole hot path of SURVEY.md §8(a) over the config's tensor:
5 HOOI sweeps + core/fit and 5 MP sweeps + core/fit (config 2 of BASELINE.json:
1000^3, 1e6 uniform nonzeros, core 50^3), each from the same seeded U0, with
the sparse tensor (CSF) already resident in HBM.  value = nonzero-mode updates
per second = nnz * N_modes * (HOOI sweeps + MP sweeps) / step time.  With N>1
(torchrun) the ranks shard the one workload (HOOI by mode-n slice ranges, MP by
slice-index ranges, NCCL allreduces inside the library):
strong scaling, time = max over ranks.

`e2e` is the same metric through the C-ABI from HOST buffers: tucker_init
(H2D + CSF build) + sweeps + core_and_fit with the core and factors copied back.
`--impl reference` times the fp64 oracle (oracle/) on the host cores on a
bounded sample (1 HOOI sweep + 1 MP sweep) of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE.json config of the timed step (default 4: the largest single-GPU config)")
    ap.add_argument("--spttmc-configs", default="1,2,3,4,5",
                    help="configs of the per-mode SpTTMc roofline table ('' to skip)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (NCCL) sweep even at N=1 (a 1-rank communicator; N>1 always shards)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "_fallback": True}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.p = None
        self.gpu = gpu_index
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out = self.p.communicate(timeout=5)[0]
        except Exception:
            self.p.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def workload(k):
    from synth import make_config
    c = make_config(k)
    c["name"] = (f"config{k}: {'x'.join(map(str, c['dims']))}, {c['nnz']} nnz ({c['kind']}), "
                 f"core {'x'.join(map(str, c['core']))}, {c['sweeps']} HOOI + {c['sweeps']} MP sweeps "
                 f"+ core/fit per step")
    return c


def compute_peaks():
    """Measured compute peaks (tools/peaks.py on a B200 of this pool, committed under
    profiles/); None where unmeasured."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "measured_compute_peaks.json")))
    except Exception:
        return {}


def spttmc_model(dims, core, layout):
    """SURVEY §8(d) algorithmic work of the HOOI SpTTMc of each mode, on the CSF
    ordering the library uses for it (tucker_csf_layout): bytes = CSF read (leaf id +
    value 8 B per nonzero, fiber id + pointer 8 B per fiber, 8 B per order-4 node) +
    Y_(n) written once in fp32 + one read of every other factor; flops = 2 J_leaf nnz
    + 2 J_mid J_leaf fibers (order 4: 2 J_mid1 J_leaf fibers + 2 J_mid0 J_mid1 J_leaf
    nodes).  Gathers served from L2 are not algorithmic bytes.  Where the library reuses a
    partial contraction (hooi_reuse_pairs) the bytes / flops are those of the path it runs:
    the root mode adds the Z write, the sibling mode is Z read once + Y written."""
    out = []
    reuse = hooi_reuse_pairs(layout)
    for n, L in enumerate(layout):
        oth = [q for q in range(len(dims)) if q != n]
        P = int(np.prod([core[q] for q in oth]))
        b = (8.0 * L["nnz"] + 8.0 * L["fibers"] + 8.0 * L["nodes"] + 4.0 * dims[n] * P
             + sum(4.0 * dims[q] * core[q] for q in oth))
        jl = core[L["leaf"]]
        if L["mid1"] < 0:
            fl = 2.0 * jl * L["nnz"] + 2.0 * core[L["mid0"]] * jl * L["fibers"]
        else:
            fl = (2.0 * jl * L["nnz"] + 2.0 * core[L["mid1"]] * jl * L["fibers"]
                  + 2.0 * P * L["nodes"])
        if n in reuse:          # root mode of a pair: also writes Z (nodes x J_mid1 J_leaf fp32)
            b += 4.0 * L["nodes"] * core[L["mid1"]] * jl
        if n - 1 in reuse:      # sibling mode: reads the kept Z once, writes Y, reads U_{n-1}
            R = layout[n - 1]
            b = (4.0 * R["nodes"] * core[R["mid1"]] * core[R["leaf"]] + 8.0 * R["nodes"] + 4.0 * dims[n] * P
                 + 4.0 * dims[n - 1] * core[n - 1])
            fl = 2.0 * P * R["nodes"]
        out.append((b, fl))
    return out


def hooi_reuse_pairs(layout):
    """Root modes p whose HOOI projection keeps Z for mode p + 1 (order 4, the library's
    partial-contraction reuse): visible in the layout as ordering (p; p + 1; x; y) for both
    p = 0 and p = 2 (no other rule produces mid0 = 3 for root 2)."""
    if len(layout) == 4 and layout[0]["mid0"] == 1 and layout[2]["mid0"] == 3:
        return (0, 2)
    return ()


def spttmc_table(capi, configs, local, stream, pk, cpk):
    """Per-config, per-mode HOOI SpTTMc time (tucker_time_ttmc: CUDA events on the
    library stream, 5 back-to-back projections after an untimed one, random U0), with
    Gnnz/s and the fractions of the HBM (measured copy bandwidth), FP32 (measured
    FFMA) and 3xTF32 (measured tcgen05 kind::tf32 issue peak / 3) rooflines."""
    import torch
    from synth import make_config
    rows = []
    hbm = pk["hbm_gbs"] * 1e9
    f32 = (cpk.get("ffma_tflops") or 148 * 128 * 2 * 1.965e9 / 1e12) * 1e12
    tf3 = ((cpk.get("tcgen05_tf32_tflops") or pk["bf16_tflops"] * 1.1 / 2.25) / 3.0) * 1e12
    for k in configs:
        c = make_config(k, device="cuda" if k == 5 else None)
        dims, core, nnz = c["dims"], c["core"], c["nnz"]
        dev = torch.device("cuda", local)
        idx = [torch.from_numpy(a).to(dev) for a in c["idx"]]
        vals = torch.from_numpy(c["vals"]).to(dev)
        U0 = [torch.from_numpy(u).to(dev) for u in c["U0"]]
        del c
        h = capi.tucker_init(dims, core, idx, vals, U0, device=local, stream=stream.cuda_stream, on_device=True)
        del idx, vals
        lay = capi.tucker_csf_layout(h, len(dims))
        model = spttmc_model(dims, core, lay)
        reuse = hooi_reuse_pairs(lay)
        for n in range(len(dims)):
            ms = capi.tucker_time_ttmc(h, n, 5)
            b, fl = model[n]
            t = ms / 1e3
            rows.append({"config": k, "mode": n + 1, "ms": round(ms, 4), "gnnz_s": nnz / t / 1e9,
                         "alg_bytes": b, "flops": fl, "hbm_frac": b / t / hbm, "fp32_frac": fl / t / f32,
                         "tf32x3_frac": fl / t / tf3,
                         "t_hbm_us": 1e6 * b / hbm, "t_fp32_us": 1e6 * fl / f32, "t_3xtf32_us": 1e6 * fl / tf3,
                         "binding": "hbm" if b / hbm >= fl / tf3 else "tensor(3xTF32)",
                         "binding_frac": max(b / hbm, fl / tf3) / t,
                         "path": ("reuse: Z kept by mode %d" % n if n - 1 in reuse else
                                  "full SpTTMc + Z kept" if n in reuse else "full SpTTMc")})
        capi.tucker_free(h)
        torch.cuda.empty_cache()
    return rows


def mp_overlap_on(c):
    """The library's MP overlap (TUCKER_MP_OVERLAP, default on; dense-W route, order >= 3):
    the main stream's projection / Gram stages then hold only the late term (m = n - 1) of
    each mode; the other terms run beside the previous mode's eigensolve."""
    # (only beside the one-CTA direct eigensolver: MP Grams of d <= 224 -- config 4, not config 2's d = 1000)
    return (os.environ.get("TUCKER_MP_OVERLAP", "1") != "0" and len(c["dims"]) >= 3 and c["nnz"] < 1e8
            and max(c["dims"]) <= 224)


def gram_flops(c, late_only=False):
    """Algorithmic flops of the Gram (SYRK, upper triangle incl. diagonal) per
    HOOI sweep and per MP sweep: d(d+1)K with d x K the Gram operand (MP: only
    the late term's K when late_only)."""
    dims, J, N = c["dims"], c["core"], len(c["dims"])
    h = m = 0.0
    for n in range(N):
        P = int(np.prod([J[q] for q in range(N) if q != n]))
        d, K = (dims[n], P) if P >= dims[n] else (P, dims[n])
        h += d * (d + 1.0) * K
        terms = [(n - 1) % N] if late_only else [q for q in range(N) if q != n]
        Kw = sum(J[q] * int(np.prod([dims[r] for r in range(N) if r not in (n, q)])) for q in terms)
        m += dims[n] * (dims[n] + 1.0) * Kw
    return h, m


def direct_eig_flops(d, J):
    """Algorithmic fp64 flops of one direct dense solve (k_eig_direct): Householder
    tridiagonalisation 4/3 d^3 (symmetric product + rank-2 update per column),
    back-transformation of J vectors 4 d^2 J / 2 (reflectors of decreasing length);
    the O(d J) bisection / inverse-iteration work is not counted."""
    return 4.0 / 3.0 * d ** 3 + 2.0 * d * d * J


def cpu_oracle_sample(c):
    """The fp64 oracle as it stands on a bounded sample: 1 HOOI sweep + 1 MP
    sweep (+ their cores) of the same workload.  Returns (seconds, units)."""
    from oracle import tucker_oracle as O
    T = O.SparseTensor(c["dims"], c["idx"], c["vals"])
    t0 = time.perf_counter()
    O.run_hooi(T, c["U0"], c["core"], 1)
    O.run_mp(T, c["U0"], c["core"], 1)
    dt = time.perf_counter() - t0
    return dt, c["nnz"] * len(c["dims"]) * 2


def host_info():
    """CPU model and BLAS library of the host the oracle runs on."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = "unknown"
    try:
        from threadpoolctl import threadpool_info
        b = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if b:
            blas = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('num_threads')} threads)"
    except Exception:
        pass
    return {"cpu_model": model, "blas": blas, "host_cores": len(os.sched_getaffinity(0))}


def cores_used():
    n = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return int(max(th))
    except Exception:
        pass
    return n


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    c = workload(args.config)
    for _ in range(args.warmup):
        cpu_oracle_sample(c)
    ts = []
    units = 0
    for _ in range(args.steps):
        dt, units = cpu_oracle_sample(c)
        ts.append(dt)
    total = sum(ts)
    val = units * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": "HOOI/MP sweep throughput (nnz x modes per second)",
        "value": val, "unit": "Gnnz/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"] + " [reference step: 1 HOOI + 1 MP sweep sample]",
                   "l2": "host oracle"},
        "cpu_baseline": {"value": val, "unit": "Gnnz/s", "cores": cores_used(), "kind": "oracle",
                         "sample": "1 HOOI sweep + 1 MP sweep (+ cores) of the workload per step"},
        "e2e": {"value": val, "unit": "Gnnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def paper_context(capi, local, stream):
    """The paper's own Table 2 run (250^3, 10 % density, J = 25) end to end through the
    C-ABI from host buffers: tucker_init (H2D + CSF build) + HO-SVD init of modes 2..N + sweeps until
    Delta_fit < 1e-4 + core_and_fit, next to the paper's whole-run MATLAB times (which include its HO-SVD init,
    sort and slice files).  Context only: one 2007 Opteron core vs one B200, different software."""
    import torch
    from synth import bernoulli_dense, random_orthonormal
    dims, core = (250, 250, 250), (25, 25, 25)
    X = bernoulli_dense(dims, 0.1, np.random.default_rng(1))
    nz = np.nonzero(X)
    idx = [np.asarray(i, dtype=np.int32) for i in nz]
    vals = X[nz].astype(np.float32)
    del X
    U0 = [random_orthonormal(I, J, np.random.default_rng(60 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    out = {"workload": "PAPER Table 2: 250^3, density 0.1 (1.56e6 nnz), core 25^3, HO-SVD init, Delta_fit < 1e-4",
           "paper_hardware": "one core of a dual-core AMD Opteron 64, MATLAB R2007a + Tensor Toolbox 2.2 (P:1159-1166)",
           "paper": {"hooi_s": 66, "hooi_fit_pct": 4.053, "mp_s": 105, "mp_fit_pct": 3.979}}
    for algo in ("hooi", "mp"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = capi.tucker_init(dims, core, idx, vals, U0, device=local, stream=stream.cuda_stream)
        capi.tucker_hosvd(h, 0b110)
        fits, _ = (capi.hooi_run if algo == "hooi" else capi.mp_run)(h, 50, 1e-4)
        _, _, fit = capi.core_and_fit(h, dims, core)
        torch.cuda.synchronize()
        out[algo + "_s"] = time.perf_counter() - t0
        out[algo + "_fit_pct"] = 100 * fit
        out[algo + "_sweeps"] = len(fits)
        capi.tucker_free(h)
    out["speedup_vs_paper"] = {a: out["paper"][a + "_s"] / out[a + "_s"] for a in ("hooi", "mp")}
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_0711_2023_b200 import capi

    c = workload(args.config)
    dims, core, N, S = c["dims"], c["core"], len(c["dims"]), c["sweeps"]
    stream = torch.cuda.current_stream(dev)
    sharded = world > 1 or args.sharded

    def nccl_id():
        """A fresh ncclUniqueId from rank 0, broadcast over torch.distributed
        (each sharded handle owns its own communicator)."""
        if not sharded:
            return {}
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(capi.nccl_unique_id()), dtype=torch.uint8))
        if world > 1:
            torch.distributed.broadcast(buf, src=0)
        return {"rank": rank, "world": world, "nccl_id": bytes(buf.cpu().numpy().tobytes())}
    idx_d = [torch.from_numpy(a).to(dev) for a in c["idx"]]
    vals_d = torch.from_numpy(c["vals"]).to(dev)
    U0_d = [torch.from_numpy(u).to(dev) for u in c["U0"]]
    G_d = torch.empty(int(np.prod(core)), dtype=torch.float32, device=dev)
    U_d = [torch.empty_like(u) for u in U0_d]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = capi.tucker_init(dims, core, idx_d, vals_d, U0_d, device=local, stream=stream.cuda_stream,
                         on_device=True, output_on_device=True, **nccl_id())
    init_s = time.perf_counter() - t0
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 512 MB > L2

    stage_acc = np.zeros(4)
    sweep_acc = np.zeros(S)      # HOOI per-sweep time (all stages), summed over timed steps
    sweep_acc_mp = np.zeros(S)
    stage_acc_mp = np.zeros(4)

    def step(record=False):
        nonlocal stage_acc, stage_acc_mp, sweep_acc, sweep_acc_mp
        capi.tucker_set_factors(h, U0_d)
        fh, sh, _ = capi.hooi_sweep(h, S, want_stage=True)
        capi.core_and_fit_into(h, G_d, U_d)
        capi.tucker_set_factors(h, U0_d)
        fm, sm, _ = capi.mp_sweep(h, S, want_fit=False, want_stage=True)
        fit_m = capi.core_and_fit_into(h, G_d, U_d)
        if record:
            stage_acc += sh.sum(axis=0)
            stage_acc_mp += sm.sum(axis=0)
            sweep_acc += sh.sum(axis=1)
            sweep_acc_mp += sm.sum(axis=1)
        return fh[-1], fit_m

    for _ in range(args.warmup):
        step()
    capi.tucker_stats(h, reset=True)
    capi.tucker_mp_overlap_times(h, reset=True)
    clk = Clocks(local) if rank == 0 else None
    times = []
    fits = None
    for _ in range(args.steps):
        flush.zero_()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fits = step(record=True)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks = clk.stop() if clk else None
    st = capi.tucker_stats(h)
    ov = capi.tucker_mp_overlap_times(h)
    total_ms = float(sum(times))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    units = c["nnz"] * N * 2 * S
    # sharded: the N ranks process the one workload together (strong scaling)
    value = units * (1 if sharded else world) / (ms_step / 1e3) / 1e9

    # ---- e2e through the C-ABI from pinned host buffers ----
    idx_h = [torch.from_numpy(a).pin_memory() for a in c["idx"]]
    vals_h = torch.from_numpy(c["vals"]).pin_memory()
    U0_h = [torch.from_numpy(u).pin_memory() for u in c["U0"]]
    G_h = torch.empty(int(np.prod(core)), dtype=torch.float32).pin_memory()
    U_h = [torch.empty(u.shape, dtype=torch.float32).pin_memory() for u in U0_h]
    h2d = sum(a.numel() * 4 for a in idx_h) + vals_h.numel() * 4 + sum(u.numel() * 4 for u in U0_h)
    d2h = G_h.numel() * 4 + sum(u.numel() * 4 for u in U_h) + 2 * 8
    # one untimed warm-up step (the first fresh handle in a process pays the memory
    # pool's one-time growth, ~80-100 ms at config 2), then the median of 5 (the host side of the
    # boxes is noisy: single samples 30-40 % above the others turn up in most runs)
    e2e_steps = 5
    e2e_ms = []
    for it in range(e2e_steps + 1):
        kw2 = nccl_id()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h2 = capi.tucker_init(dims, core, [a.numpy() for a in idx_h], vals_h.numpy(),
                              [u.numpy() for u in U0_h], device=local, stream=stream.cuda_stream, **kw2)
        capi.hooi_sweep(h2, S)
        capi.core_and_fit_into(h2, G_h.numpy(), [u.numpy() for u in U_h])
        capi.tucker_set_factors(h2, [u.numpy() for u in U0_h])
        capi.mp_sweep(h2, S, want_fit=False)
        capi.core_and_fit_into(h2, G_h.numpy(), [u.numpy() for u in U_h])
        e1.record(stream)
        torch.cuda.synchronize()
        capi.tucker_free(h2)
        if it > 0:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_med = statistics.median(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_med], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_med = float(t.item())
    e2e_val = units / (e2e_med / 1e3) / 1e9 * (1 if sharded else world)

    # ---- roofline of the dominant kernel ----
    pk = peaks()
    cpk = compute_peaks()
    shares = {"spttmc": stage_acc[0] / args.steps, "spmm": stage_acc_mp[0] / args.steps,
              "gram": (stage_acc[1] + stage_acc_mp[1]) / args.steps,
              "eig": (stage_acc[2] + stage_acc_mp[2]) / args.steps,
              "core+fit": (stage_acc[3] + stage_acc_mp[3]) / args.steps}
    # HOOI solves: the warm-started fused solver (k_eig_fused, its own flop count); MP solves at
    # d <= 224: the one-CTA direct solver (k_eig_direct, direct_eig_flops)
    eig_ms_h = stage_acc[2] / args.steps
    eig_ms_m = stage_acc_mp[2] / args.steps
    eig_flops = st.get("eig_flops", 0) / args.steps
    launches_eig = N * S  # one launch per factor update
    fp64_peak = cpk.get("dmma_tflops") or 148 * 64 * 2 * 1.965e9 / 1e12
    peak_note = ("fp64 DMMA measured (tools/peaks.cu, profiles/measured_compute_peaks.json)"
                 if cpk.get("dmma_tflops") else
                 "fp64 nominal: 148 SMs x 64 FMA/clk x 2 x 1.965 GHz (B200_PROFILING clock)")
    try:  # per-launch DRAM bytes from the committed ncu --set full captures
        traffic_all = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        traffic_all = {}
    ach_h = eig_flops / (eig_ms_h / 1e3) / 1e12 if eig_ms_h > 0 else 0.0
    roof_eig_h = {"kernel": "k_eig_fused (HOOI: persistent warm-started subspace iteration, 32 CTAs at d <= 256)",
                  "bound": "alu", "peak_note": peak_note,
                  "achieved": ach_h, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach_h / fp64_peak,
                  "traffic": traffic_all.get("k_eig_fused"), "flops_per_launch": eig_flops / launches_eig,
                  "ms_per_launch": eig_ms_h / launches_eig, "launches_per_step": launches_eig,
                  "products_per_solve": st.get("eig_matvec", 0) / args.steps / launches_eig}
    # MP overlap: kernel time per stream from the library's events (tucker_mp_overlap_times); the
    # main-stream stage timers above then hold waits on the other streams, not kernel time
    ovl = mp_overlap_on(c) and ov["eig"][1] > 0
    terms_step = S * N * (N - 1)          # k_spmm_w launches per step (one per term)
    if ovl:
        def per_step(keys, expected):    # scale for the calls not counted (a call's last side work)
            ms = sum(ov[k][0] for k in keys)
            cnt = sum(ov[k][1] for k in keys)
            return ms / cnt * expected if cnt else 0.0
        spmm_ms_step = per_step(("side_spmm", "main_spmm"), terms_step)
        gram_mp_ms_step = (per_step(("side_gram",), S * N) + per_step(("main_gram",), S * N))
        eig_ms_m = per_step(("eig",), S * N)
    else:
        spmm_ms_step = stage_acc_mp[0] / args.steps
        gram_mp_ms_step = stage_acc_mp[1] / args.steps
    dflops = sum(direct_eig_flops(dims[n], core[n]) for n in range(N)) * S
    ach_m = dflops / (eig_ms_m / 1e3) / 1e12 if eig_ms_m > 0 else 0.0
    roof_eig = {"kernel": "k_eig_direct (MP: one-CTA dense solve -- Householder tridiagonalisation in shared "
                          "memory, multisection, inverse iteration, back-transformation)",
                "bound": "alu", "peak_note": peak_note + "; the kernel runs on ONE SM by design (beside the "
                "overlapped next-mode work on the other 147): frac_one_sm is against 1/148 of that peak",
                "achieved": ach_m, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach_m / fp64_peak,
                "frac_one_sm": ach_m / (fp64_peak / 148.0),
                "traffic": traffic_all.get("k_eig_direct"), "flops_per_launch": dflops / launches_eig,
                "ms_per_launch": eig_ms_m / launches_eig, "launches_per_step": launches_eig,
                "note": "latency bound: 198 dependent Householder steps (three block barriers each) at d = 200"}
    phases = {k: v / args.steps for k, v in st.get("eig_phase_ms", {}).items()}
    if any(v > 0 for v in phases.values()):  # only in TK_EIG_PROFILE builds (tools/eig_profile.sh)
        roof_eig["eig_phase_ms_per_step"] = phases
    # the Gram SYRK: 3xTF32 on tcgen05 (MP) / fp64 DMMA (HOOI <= 2e10 FMA)
    hflops, mflops = gram_flops(c, late_only=False)
    gram_ms = stage_acc[1] / args.steps + gram_mp_ms_step
    gram_flops_step = S * (hflops + mflops)
    g_ach = gram_flops_step / (gram_ms / 1e3) / 1e12 if gram_ms > 0 else 0.0
    tf32_peak = cpk.get("tcgen05_tf32_tflops") or pk["bf16_tflops"] * (1.1 / 2.25)
    g_peak = tf32_peak / 3.0
    roof_gram = {"kernel": "k_syrk_tc (tcgen05 3xTF32 SYRK, fp64 drain) + k_syrk_dmma", "bound": "tensor",
                 "note": ("all Grams: HOOI's, and MP's side-stream (early terms) + main-stream (late term) "
                          "kernel time" if ovl else "all Grams"),
                 "ms_per_step": gram_ms,
                 "peak_note": ("measured tcgen05 kind::tf32 issue peak / 3 products (profiles/measured_compute_peaks.json)"
                               if cpk.get("tcgen05_tf32_tflops") else
                               "measured bf16 burst x tf32/bf16 nominal (1.1/2.25) / 3 products"),
                 "achieved": g_ach, "peak": g_peak, "unit": "TFLOP/s", "frac": g_ach / g_peak}
    # HOOI SpTTMc of the timed workload (per sweep, all modes): §8(d) bytes / flops
    layout = capi.tucker_csf_layout(h, N)
    model = spttmc_model(dims, core, layout)
    hooi_proj_ms = stage_acc[0] / args.steps / S
    sp_bytes = sum(b for b, _ in model)
    sp_flops = sum(f for _, f in model)
    roof_sp = {"kernel": "k_spttmc3/k_spttmc4 (HOOI SpTTMc, all modes of one sweep)",
               "reuse": ("modes 2 and 4 from the Z kept by modes 1 and 3 (k_spttmc4_sib); bytes / flops of "
                         "the path run" if hooi_reuse_pairs(layout) else None),
               "bound": "hbm", "unit": "GB/s",
               "achieved": sp_bytes / (hooi_proj_ms / 1e3) / 1e9 if hooi_proj_ms > 0 else None,
               "peak": pk["hbm_gbs"], "alg_bytes": sp_bytes, "flops": sp_flops,
               "ms_per_sweep": hooi_proj_ms,
               "gnnz_s_per_mode": c["nnz"] * N / (hooi_proj_ms / 1e3) / 1e9 if hooi_proj_ms > 0 else None,
               "traffic": traffic_all.get("k_spttmc4" if N == 4 else "k_spttmc3")}
    roof_sp["frac"] = roof_sp["achieved"] / roof_sp["peak"] if roof_sp["achieved"] else None
    # MP's leaf SpMM (k_spmm_w): algorithmic bytes = CSF read (8 B per nonzero, 16 B per fiber incl. its
    # coordinates) + W written once (hi + lo tf32 pair, 8 B per present entry) per term
    sp_nnz_bytes = 0.0
    for n in range(N):
        for m in range(N):
            if m != n:
                sp_nnz_bytes += 8.0 * c["nnz"] + 16.0 * layout[n]["fibers"] + 8.0 * layout[n]["fibers"] * core[m]
    spmm_ms = spmm_ms_step / S
    roof_spmm = {"kernel": "k_spmm_w (MP leaf SpMM into the K-tile-major W)", "bound": "hbm", "unit": "GB/s",
                 "achieved": sp_nnz_bytes / (spmm_ms / 1e3) / 1e9 if spmm_ms > 0 else None, "peak": pk["hbm_gbs"],
                 "alg_bytes": sp_nnz_bytes, "ms_per_sweep": spmm_ms,
                 "bytes_per_launch": sp_nnz_bytes / (N * (N - 1)), "ms_per_launch": spmm_ms / (N * (N - 1)),
                 "launches_per_step": terms_step,
                 "traffic": traffic_all.get("k_spmm_w"),
                 "note": "one launch per MP term (n, m); fibers of the (n, o, m) orderings approximated by the "
                         "HOOI ordering's fiber count" +
                         ("; kernel time of the side-stream (early terms) and main-stream (late term) launches "
                          "from the library's events (tucker_mp_overlap_times)" if ovl else "")}
    roof_spmm["frac"] = roof_spmm["achieved"] / roof_spmm["peak"] if roof_spmm["achieved"] else None
    # dominant kernel: by kernel time per step (under the MP overlap the streams run side by side, so
    # the kernel times sum to more than the step; the ncu launch list gives the same ranking)
    kern = {"spttmc": stage_acc[0] / args.steps, "spmm": spmm_ms_step, "gram": gram_ms,
            "eig_hooi": eig_ms_h, "eig_mp": eig_ms_m,
            "core+fit": (stage_acc[3] + stage_acc_mp[3]) / args.steps}
    dom = max(kern, key=kern.get)
    roof = dict({"spttmc": roof_sp, "spmm": roof_spmm, "gram": roof_gram, "eig_mp": roof_eig,
                 "eig_hooi": roof_eig_h}.get(dom, roof_eig))
    roof["dominant_stage"] = dom
    roof["kernel_ms_per_step"] = kern
    roof["kernel_ms_note"] = ("per-kernel-family time per step; MP's SpMM / Gram / eigensolve run on three "
                              "streams side by side (mp_overlap), so the sum exceeds ms_per_step"
                              if ovl else "main-stream stage timers")
    roof["main_stream_stage_ms_per_step"] = shares

    line = {
        "metric": "HOOI/MP sweep throughput (nnz x modes per second)",
        "value": value, "unit": "Gnnz/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "f32+3xtf32+f64",
        "dtype_detail": "mixed: fp32 storage and SpTTMc/SpMM arithmetic; Gram products 3xTF32 on tcgen05 (MP) or "
                        "fp64 DMMA (HOOI Grams <= 2e10 FMA), both accumulated in fp64; fp64 eigensolver, core "
                        "accumulation and fit",
        "data": "synthetic",
        "config": {"workload": c["name"], "l2": "flushed (512 MB write) before every timed step",
                   "parallelism": (f"sharded x{world}: HOOI by mode-n slice ranges, MP by slice-index ranges; "
                                   "NCCL allreduce of Y / partial Gram / U / G / M_n (DESIGN.md Multi-GPU)")
                   if sharded else "single GPU"},
        "hooi_ms_per_sweep": float(stage_acc.sum() / args.steps / S),
        # sweep 0 (cold eigensolves from U0) apart from the warm sweeps >= 1
        "sweep_ms": {"hooi_sweep0": float(sweep_acc[0] / args.steps),
                     "hooi_sweeps_ge1": float(sweep_acc[1:].mean() / args.steps) if S > 1 else None,
                     "mp_sweep0": float(sweep_acc_mp[0] / args.steps),
                     "mp_sweeps_ge1": float(sweep_acc_mp[1:].mean() / args.steps) if S > 1 else None},
        "mp_ms_per_sweep": float(stage_acc_mp.sum() / args.steps / S),
        "fit": {"hooi": fits[0], "mp": fits[1]},
        "csf_build_s": init_s,
        "gpu_launches": int(st["launches"]) // args.steps,
        "gpu_launches_note": "library kernel launches per step (tucker_stats)",
        "e2e": {"value": e2e_val, "unit": "Gnnz/s", "ms_samples": [round(float(v), 3) for v in e2e_ms],
                "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "roofline": roof,
        "roofline_eig": roof_eig,
        "roofline_eig_hooi": roof_eig_h,
        "mp_overlap": ovl,
        "roofline_gram": roof_gram,
        "roofline_spttmc": roof_sp,
        "roofline_spmm": roof_spmm,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, u = cpu_oracle_sample(c)
        line["cpu_baseline"] = {"value": u / dt / 1e9, "unit": "Gnnz/s", "cores": cores_used(),
                                "kind": "oracle", "seconds": dt, **host_info(),
                                "sample": "1 HOOI sweep + 1 MP sweep (+ cores) of the same workload"}
    capi.tucker_free(h)
    if rank == 0 and world == 1 and args.spttmc_configs:
        del idx_d, vals_d
        torch.cuda.empty_cache()
        line["spttmc_table"] = spttmc_table(capi, [int(x) for x in args.spttmc_configs.split(",")], local,
                                            stream, pk, cpk)
    if rank == 0 and world == 1:
        line["paper_context"] = paper_context(capi, local, stream)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
