"""Benchmark: Shampoo optimizer step on the ResNet-50 parameter set (BASELINE.json configs 2/3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--precision double|single] [--workload resnet50|mlp|vit_b_16|gpt2_medium]
    python bench.py --sweep rootinv      # BASELINE config 5: root-inverse ms/block, eigh vs Newton

One process per GPU (NCCL).  ``--gpus N`` with N > 1 outside torchrun re-launches
itself under ``torch.distributed.run`` (one rank per GPU, 127.0.0.1 rendezvous).

A "step" is one full optimizer step over the 161 ResNet-50 parameter tensors
(25.56 M variables) with synthetic fp32 gradients resident in HBM: statistics,
root inverse when t % f == 0 (f = 50), preconditioning + grafting + momentum,
all-gather of the directions (N > 1), parameter update.

Steady state.  Before any timing the optimizer is fast-forwarded to step T0
(default 2600, past the point where every 2048-dim vector factor is full rank):
the factor statistics of T0 - f steps are accumulated from fresh gradients
(statistics only -- with synthetic gradients the factors do not depend on the
parameters, so they equal those of full steps), then f full steps (one refresh)
run, then the timed window starts AT a refresh step.  Each timed step is
bracketed by CUDA events on the launching stream; the amortised step over one
precondition cycle is

    value = ((f - 1) * mean(plain steps) + mean(refresh steps)) / f

which is what a training run pays per step.  The window's raw mean is reported
beside it.  W >= 3 extra warm-up steps precede the fast-forward.  The optimizer
state (factors + inverses ~2 GB) is far larger than the 126 MB L2, so no flush.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy oracle port of minishampoo, oracle/shampoo_oracle.py) on the host cores
with every thread the BLAS can use, on a bounded sample (cpu_baseline.sample).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Shampoo step ms (ResNet-50 params) at 1/2/4/8 B200; root-inverse ms/block"

# per workload: shapes key, ShampooConfig kwargs (BASELINE.json configs)
COMMON = dict(precondition_frequency=50, betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True,
              weight_decay=1e-4, use_decoupled_weight_decay=True)
WORKLOADS = {
    "resnet50": dict(max_preconditioner_dim=2048, grafting="adagrad"),
    "mlp": dict(max_preconditioner_dim=512, grafting="adagrad"),
    "vit_b_16": dict(max_preconditioner_dim=1024, grafting="adam"),
    "gpt2_medium": dict(max_preconditioner_dim=1024, grafting="adam"),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1370.0,
         "source": "fallback (B200_PROFILING.md)"}
    if os.path.exists(path):
        d = json.load(open(path))
        p.update(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"],
                 bf16_tflops_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                 source="measured (MEASURED_PEAKS.json)")
    fp64 = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(fp64):
        p["fp64_tflops"] = json.load(open(fp64))["fp64_tflops"]
    return p


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def model_shapes(workload: str):
    from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
    return [tuple(s) for s in MODEL_SHAPES[workload]]


def amortise(step_ms, is_refresh, f):
    """((f-1) * mean(plain) + mean(refresh)) / f from per-step times of one window."""
    plain = [m for m, r in zip(step_ms, is_refresh) if not r]
    refr = [m for m, r in zip(step_ms, is_refresh) if r]
    p = float(np.mean(plain)) if plain else None
    r = float(np.mean(refr)) if refr else None
    if p is None:
        return r, p, r
    if r is None:
        return p, p, r
    return ((f - 1) * p + r) / f, p, r


# ---------------------------------------------------------------- reference (CPU) arm


def cpu_reference(workload: str, sample_plain_steps: int = 1, rootinv_budget_s: float = 8.0):
    """Oracle (numpy float64, reference algorithm) on the full parameter set of the workload.

    Sample: `sample_plain_steps` non-refresh steps over every block (preset inverses so the full
    preconditioning path runs) plus eigh root inverses of full-rank synthetic factors for the
    distinct factor sizes (largest first, within a time budget), scaled by sum n^3 to the full
    refresh; amortised = plain + refresh / f.  A lower bound on the reference: it skips the
    reference's per-call symmetry/finiteness checks and the refresh-step bookkeeping.
    """
    from oracle import shampoo_oracle as O

    shapes = model_shapes(workload)
    wl = WORKLOADS[workload]
    f = COMMON["precondition_frequency"]
    rng = np.random.default_rng(0)
    params = [(rng.standard_normal(s) * 0.05).astype(np.float32).astype(np.float64) for s in shapes]
    grng = np.random.default_rng(1)
    kw = dict(COMMON, max_preconditioner_dim=wl["max_preconditioner_dim"])
    cfg = O.OracleConfig(grafting=O.GraftKind(wl["grafting"]), **kw)
    opt = O.OracleShampoo(params, cfg)
    opt.t = 1  # a non-refresh step; preset inverses = I so precondition runs
    sizes = {}
    for row in opt.states:
        for st in row:
            if st is not None and st.kind == "shampoo":
                st.inverses = [np.eye(d) for d in st.shape]
                for d in st.shape:
                    sizes[(d, 2 * len(st.shape))] = sizes.get((d, 2 * len(st.shape)), 0) + 1
    plain = []
    for _ in range(sample_plain_steps):
        grads = [(grng.standard_normal(s) * 1e-2).astype(np.float32).astype(np.float64) for s in shapes]
        t0 = time.perf_counter()
        opt.step(grads)
        plain.append(time.perf_counter() - t0)
        opt.t = 1
    refresh_s, measured_n3 = 0.0, 0.0
    total_n3 = sum(c * d ** 3 for (d, _), c in sizes.items())
    spent = 0.0
    per_size = {}
    for d, p in sorted(sizes, reverse=True):
        if d in per_size:
            continue
        g = rng.standard_normal((d, 2 * d))
        a = g @ g.T / (2 * d) + 1e-3 * np.eye(d)
        t0 = time.perf_counter()
        O.root_inverse_eigh(a, p, eps=1e-12)
        dt = time.perf_counter() - t0
        per_size[d] = dt
        spent += dt
        if spent > rootinv_budget_s:
            break
    for (d, _), c in sizes.items():
        if d in per_size:
            refresh_s += c * per_size[d]
            measured_n3 += c * d ** 3
    refresh_s *= total_n3 / max(measured_n3, 1.0)
    plain_ms = 1e3 * float(np.median(plain))
    amort_ms = plain_ms + 1e3 * refresh_s / f
    ndist = len({d for d, _ in sizes})
    return {"plain_ms": plain_ms, "refresh_extra_ms": 1e3 * refresh_s, "amortized_ms": amort_ms,
            "cores": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count())),
            "sample": (f"{sample_plain_steps} plain step(s) over all {len(shapes)} {workload} tensors (oracle port "
                       f"of minishampoo, float64) + eigh root inverses of {len(per_size)}/{ndist} distinct factor "
                       f"sizes scaled by sum n^3 to the full refresh; amortised over f={f}; lower bound on the "
                       "reference (no per-call symmetry checks)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    steps = max(1, min(args.steps, 2))
    r = cpu_reference(args.workload, sample_plain_steps=steps)
    wl = WORKLOADS[args.workload]
    line = {"metric": METRIC, "value": round(r["amortized_ms"], 3), "unit": "ms", "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": 0,
            "ms_per_step": round(r["amortized_ms"], 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}_shampoo_step", "max_preconditioner_dim": wl["max_preconditioner_dim"],
                       "precondition_frequency": COMMON["precondition_frequency"], "grafting": wl["grafting"],
                       "parallelism": "cpu (the reference has no parallel multi-rank path: J=1 CPU is the "
                                      "baseline for every N)"},
            "cpu_baseline": {"value": round(r["amortized_ms"], 3), "unit": "ms", "cores": r["cores"],
                             "kind": "port", "sample": r["sample"], "plain_ms": round(r["plain_ms"], 1),
                             "refresh_ms": round(r["refresh_extra_ms"], 1)},
            "e2e": {"value": round(r["amortized_ms"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2309_06497_b200 as P
    from paper_2309_06497_b200 import _native as N
    from paper_2309_06497_b200.distributed import GroupExchange
    import ctypes as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS[args.workload]
    shapes = model_shapes(args.workload)
    numels = [math.prod(s) for s in shapes]
    n_params = sum(numels)
    f = COMMON["precondition_frequency"]
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    params = [torch.randn(s, generator=gen, device=dev) * 0.05 for s in shapes]
    # identical gradients on every rank (the reference models no gradient all-reduce, dist.py:332-356)
    gen.manual_seed(1)
    flat = torch.empty(n_params, device=dev)

    def fresh():
        """One fresh N(0, 0.01^2) fp32 gradient set (views of one flat buffer)."""
        torch.randn(n_params, generator=gen, device=dev, out=flat)
        flat.mul_(1e-2)
        return [v.view(s) for v, s in zip(torch.split(flat, numels), shapes)]

    def resident(k):
        """k fresh gradient sets resident in HBM for one timed window: all distinct when they fit in
        8 GB (ResNet-50: 0.1 GB each), else as many as fit, used cyclically (GPT-2-medium: 1.4 GB
        each; at the steady state every factor is full rank, so reuse changes no work)."""
        nd = max(2, min(k, int(8e9 // (4 * n_params))))
        out = []
        for _ in range(nd):
            g = fresh()
            out.append([x.clone() for x in g])
        return [out[i % nd] for i in range(k)]

    cfg = P.ShampooConfig(grafting=P.GraftKind(wl["grafting"]), precision=args.precision,
                          max_preconditioner_dim=wl["max_preconditioner_dim"], **COMMON)
    exchange = GroupExchange(world) if world > 1 else None
    opt = P.Shampoo(params, cfg, world_size=world, group_size=world, rank=rank, exchange=exchange,
                    check_finite="deferred" if args.check_finite == "deferred" else True)
    lib = N.lib()
    stream = torch.cuda.current_stream(dev)
    pdt = N.DTYPE_F32
    pp = N.ptr_array([p.data_ptr() for p in params])

    def is_refresh(t):
        return t >= cfg.start_preconditioning_step and t % f == 0

    # ---- warm-up + fast-forward to the steady state
    t_start = time.perf_counter()
    for _ in range(args.warmup):
        opt.step(fresh())
    T0 = args.steady_step
    if T0 < 0:
        T0 = int(math.ceil(1.25 * wl["max_preconditioner_dim"] / f)) * f
    T0 = max(T0, int(math.ceil((opt.step_count + f) / f)) * f)
    # statistics only up to T0 - f (factors do not depend on the parameters under synthetic gradients)
    while opt.step_count < T0 - f:
        g = fresh()
        gp = N.ptr_array([x.data_ptr() for x in g])
        N.check(lib.shampoo_stats_update(opt._ctx, gp, pp, pdt, opt.step_count, stream.cuda_stream), "ff")
        opt.advance_step()
    while opt.step_count < T0:  # one full precondition cycle (refresh at T0 - f)
        opt.step(fresh())
    torch.cuda.synchronize()
    ff_s = time.perf_counter() - t_start

    def to_refresh():
        while not is_refresh(opt.step_count):
            opt.step(fresh())

    def window(grads, timed_phases=False, exch=None):
        """K steps from the current (refresh) step; per-step CUDA events on the launching stream."""
        lib.shampoo_timing_enable(opt._ctx, 1 if timed_phases else 0)
        lib.shampoo_timing_get(opt._ctx, None, None)
        if exch is not None:
            opt.exchange = exch
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        refresh = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = P.launch_count()
        h0 = time.perf_counter()
        ev[0].record(stream)
        enq = []
        for k in range(args.steps):
            refresh.append(is_refresh(opt.step_count))
            e0 = opt.host_enqueue_s
            opt.step(grads[k])
            enq.append(opt.host_enqueue_s - e0)
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
        host_s = time.perf_counter() - h0
        window.enqueue_ms = [1e3 * x for x in enq]
        opt.exchange = exchange
        per = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
        return per, refresh, ev[0].elapsed_time(ev[-1]), host_s, P.launch_count() - l0

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor([v if v is not None else -1.0 for v in vals], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) if x >= 0 else None for x in t.tolist()]

    # ---- 1) the timed window (no per-phase instrumentation)
    grads = resident(args.steps)
    lib.shampoo_tc_counter(1, None)
    prof = os.environ.get("SHAMPOO_BENCH_PROFILE") == "1"  # ncu --profile-from-start off: this window only
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    with Clocks(local) as clk:
        per, refr, total_ms, host_s, launches = window(grads)
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    value, plain_ms, refresh_ms = amortise(per, refr, f)
    enq_plain = [m for m, r in zip(window.enqueue_ms, refr) if not r]
    host_enqueue_ms = float(np.median(enq_plain)) if enq_plain else None
    value, plain_ms, refresh_ms, total_ms = max_over_ranks([value, plain_ms, refresh_ms, total_ms])
    window_ms = total_ms / args.steps

    # ---- 2) per-phase window (starts at the next refresh), exchange timed on the stream
    to_refresh()
    gather_ev = []

    def timed_exchange(buf, gr, mp):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        exchange(buf, gr, mp)
        b.record(stream)
        gather_ev.append((a, b))

    del grads
    grads = resident(args.steps)
    torch.cuda.synchronize()
    lib.shampoo_tc_counter(1, None)
    lib.shampoo_gemm_timing(1, None, None, None)  # reset + bracket every tensor-core GEMM launch
    pper, prefr, _, _, _ = window(grads, timed_phases=True, exch=timed_exchange if exchange else None)
    ozw = C.c_double()
    lib.shampoo_tc_counter(0, C.byref(ozw))
    gk_ms, gk_ops, gk_n = (C.c_double * 8)(), (C.c_double * 8)(), (C.c_int64 * 8)()
    lib.shampoo_gemm_timing(0, gk_ms, gk_ops, gk_n)
    ms = (C.c_double * 5)()
    cnt = (C.c_int64 * 5)()
    lib.shampoo_timing_get(opt._ctx, ms, cnt)
    lib.shampoo_timing_enable(opt._ctx, 0)
    names = ["stats", "root_inverse", "precondition", "graft_momentum", "apply"]
    per_call = {k: (ms[i] / cnt[i] if cnt[i] else 0.0) for i, k in enumerate(names)}
    gather_ms = (sum(a.elapsed_time(b) for a, b in gather_ev) / len(gather_ev)) if gather_ev else 0.0
    n_refresh = sum(prefr)
    phase_vals = max_over_ranks([per_call[k] for k in names] + [gather_ms])
    per_call = dict(zip(names, phase_vals[:5]))
    gather_ms = phase_vals[5]
    phase_ms = {"stats": per_call["stats"], "precondition": per_call["precondition"],
                "graft_momentum": per_call["graft_momentum"], "apply": per_call["apply"],
                "root_inverse_per_refresh": per_call["root_inverse"],
                "root_inverse_amortized": per_call["root_inverse"] / f, "allgather": gather_ms}

    # ---- roofline: tensor pipe (int8 tcgen05) for the GEMM phases and the refresh, HBM for the rest
    pk = peaks()
    int8_peak = 2.0 * pk["bf16_tflops"]  # B200 dense int8 = 2 x dense bf16; bf16 measured (burst)
    sf, pf, n3 = C.c_double(), C.c_double(), C.c_double()
    lib.shampoo_work(opt._ctx, C.byref(sf), C.byref(pf), C.byref(n3))
    so, po, stf, ptf = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    lib.shampoo_work_tc(opt._ctx, C.byref(so), C.byref(po), C.byref(stf), C.byref(ptf))
    # int8 ops executed in the phase window: plain-step GEMMs (known per step) + the refresh's GEMMs
    steps_w = args.steps
    refresh_int8 = max(ozw.value - steps_w * (so.value + po.value), 0.0) / max(n_refresh, 1)
    n_el = n_params
    esz = 8 if args.precision == "double" else 4

    def tc_kernel(ops, flops64, ms_):
        a = ops / (ms_ * 1e-3) / 1e12 if ms_ else 0.0
        return {"bound": "tensor", "achieved": round(a, 1), "peak": round(int8_peak, 1), "unit": "TOPS (int8)",
                "frac": round(a / int8_peak, 4), "ms": round(ms_, 4),
                "fp64_equivalent_tflops": round(flops64 / (ms_ * 1e-3) / 1e12, 2) if ms_ else None,
                "tensor_core": "tcgen05.mma kind::i8 (Ozaki split, exact int32 accumulation)"}

    kernels = {
        "stats_gemm": tc_kernel(so.value, sf.value, per_call["stats"]),
        "precondition_gemm": tc_kernel(po.value, pf.value, per_call["precondition"]),
    }
    kernels["stats_gemm"]["work"] = f"{sf.value/1e9:.2f} GFLOP FP64-class = {so.value/1e12:.2f} int8 Tops executed"
    kernels["precondition_gemm"]["work"] = f"{pf.value/1e9:.2f} GFLOP FP64-class = {po.value/1e12:.2f} int8 Tops executed"
    if per_call["root_inverse"]:
        ri = tc_kernel(refresh_int8, 9.0 * n3.value, per_call["root_inverse"])
        ri.update(ms_per_refresh=round(per_call["root_inverse"], 2),
                  work=f"{refresh_int8/1e12:.1f} int8 Tops executed per refresh (device counter); "
                       f"sum n^3 = {n3.value/1e9:.1f} G",
                  note="steady-state refresh: coupled-Newton pre-pass GEMMs on the tcgen05 Ozaki engine (+ "
                       "power iterations, residual checks); fp64_equivalent counts a tridiagonal eigh (9 n^3)")
        kernels["root_inverse"] = ri
    besz = opt.gather_buffer.element_size()  # float32 directions for float32 parameters
    graft_bytes = n_el * (esz * 3 + 4 + besz)  # P_sh read, momentum r/w, fp32 W read (WD), direction write
    apply_bytes = n_el * (besz + 8)            # direction read + fp32 W read/write
    for k, b in (("graft_momentum", graft_bytes), ("apply", apply_bytes)):
        m = per_call[k]
        a = b / (m * 1e-3) / 1e9 if m else 0.0
        kernels[k] = {"bound": "hbm", "achieved": round(a, 1), "unit": "GB/s", "peak": pk["hbm_gbs"],
                      "frac": round(a / pk["hbm_gbs"], 4), "ms": round(m, 4), "bytes": b}
    if world > 1:
        gbytes = (world - 1) * opt.max_payload * opt.gather_buffer.element_size()
        a = gbytes / (gather_ms * 1e-3) / 1e9 if gather_ms else 0.0
        kernels["allgather"] = {"bound": "nvlink", "achieved": round(a, 1), "unit": "GB/s (received per rank)",
                                "peak": 900.0, "frac": round(a / 900.0, 4), "ms": round(gather_ms, 4),
                                "bytes_per_rank": gbytes, "peak_source": "NVLink 5 nominal, per direction"}
    amort = {"stats": per_call["stats"], "precondition": per_call["precondition"],
             "root_inverse": per_call["root_inverse"] / f}
    dom = max(amort, key=amort.get)
    dk = {"stats": "stats_gemm", "precondition": "precondition_gemm", "root_inverse": "root_inverse"}[dom]
    if dk not in kernels:
        dk = "precondition_gemm"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload, {}).get(dk)
    # kernel level: the k_oz_gemm_p launches of each phase alone (CUDA events around every launch,
    # executed int8 ops counted on the device per phase) -- the roofline the contract asks for
    for key, tag in (("stats_gemm", 0), ("root_inverse", 1), ("precondition_gemm", 2)):
        if key in kernels and gk_n[tag] and gk_ms[tag] > 0:
            a = gk_ops[tag] / (gk_ms[tag] * 1e-3) / 1e12
            kernels[key]["kernel_level"] = {
                "kernel": "k_oz_gemm_p (tcgen05.mma kind::i8)", "achieved": round(a, 1), "unit": "TOPS (int8)",
                "frac": round(a / int8_peak, 4), "launches": int(gk_n[tag]),
                "ms_per_launch": round(gk_ms[tag] / gk_n[tag], 4), "int8_tops_executed": round(gk_ops[tag] / 1e12, 3),
                "window": f"{args.steps} steps incl. {n_refresh} refresh"}
    kl = kernels[dk].get("kernel_level")
    roofline = {"bound": "tensor", "kernel": (dk + " / k_oz_gemm_p") if kl else dk,
                "achieved": kl["achieved"] if kl else kernels[dk]["achieved"], "peak": kernels[dk]["peak"],
                "unit": "TOPS (int8)", "frac": kl["frac"] if kl else kernels[dk]["frac"],
                "phase_achieved": kernels[dk]["achieved"], "phase_frac": kernels[dk]["frac"], "traffic": traffic,
                "peak_source": "2 x measured dense bf16 burst (MEASURED_PEAKS.json; B200 int8:bf16 = 2:1)",
                "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()}, "kernels": kernels,
                "sum_n3_G": round(n3.value / 1e9, 2)}

    # ---- 3) e2e through the public API with host buffers, starting at the next refresh: every step's
    # gradients H2D from pinned host memory and every step's parameters D2H.  Pipelined like a data
    # loader: NB gradient buffers (the H2D of step k may start once step k - NB finished reading its
    # buffer) and two parameter snapshots (the D2H of step k overlaps steps k+1, k+2); all copies
    # complete inside the window
    e2e = None
    if not args.skip_e2e:
        to_refresh()
        del grads
        host_grads = [torch.cat([x.reshape(-1) for x in fresh()]).cpu().pin_memory() for _ in range(args.steps)]
        host_params = torch.empty(n_params, dtype=torch.float32).pin_memory()
        NB = 3
        dev_flat = [torch.empty(n_params, dtype=torch.float32, device=dev) for _ in range(NB)]
        dev_grads = [[v.view(s_) for v, s_ in zip(torch.split(fl, numels), shapes)] for fl in dev_flat]
        snap_flat = [torch.empty(n_params, dtype=torch.float32, device=dev) for _ in range(2)]
        snap = [[v.view(s_) for v, s_ in zip(torch.split(fl, numels), shapes)] for fl in snap_flat]
        h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(NB)]
        ev_used = [torch.cuda.Event() for _ in range(NB)]
        ev_snap = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        erefr = []
        # warm the copy machinery outside the window (first-use costs -- lazy kernel-module loading of the
        # multi-tensor snapshot copy, first DMA to each pinned buffer -- would otherwise land in the
        # window's first step, which is the refresh step: +14 ms measured)
        for q in range(2):
            torch._foreach_copy_(snap[q], list(opt.params()))
            host_params.copy_(snap_flat[q], non_blocking=True)
        for b in range(NB):
            dev_flat[b].copy_(host_grads[b % len(host_grads)], non_blocking=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)

        def upload(k):
            b = k % NB
            with torch.cuda.stream(h2d):
                h2d.wait_event(ev[0])
                if k >= NB:
                    h2d.wait_event(ev_used[b])  # step k - NB finished reading this buffer
                dev_flat[b].copy_(host_grads[k], non_blocking=True)
                ev_in[b].record(h2d)

        for k in range(min(NB - 1, args.steps)):
            upload(k)
        for k in range(args.steps):
            b, q = k % NB, k % 2
            if k + NB - 1 < args.steps:
                upload(k + NB - 1)
            erefr.append(is_refresh(opt.step_count))
            stream.wait_event(ev_in[b])
            opt.step(dev_grads[b])
            ev_used[b].record(stream)
            if k >= 2:
                stream.wait_event(ev_out[q])  # the read-back of step k-2 finished with this snapshot
            torch._foreach_copy_(snap[q], list(opt.params()))  # device snapshot (D2D), read back below
            ev_snap[q].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_snap[q])
                host_params.copy_(snap_flat[q], non_blocking=True)
                ev_out[q].record(d2h)
            if k + 1 == args.steps:
                stream.wait_event(ev_out[q])
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
        eper = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
        e_val, e_plain, e_refr = amortise(eper, erefr, f)
        e_val, e_plain, e_refr = max_over_ranks([e_val, e_plain, e_refr])
        e2e = {"value": round(e_val, 3), "unit": "ms", "h2d_bytes_per_step": 4 * n_params,
               "d2h_bytes_per_step": 4 * n_params, "steps": args.steps, "refresh_steps": sum(erefr),
               "plain_ms": round(e_plain, 3) if e_plain else None,
               "refresh_ms": round(e_refr, 3) if e_refr else None,
               "note": "Shampoo.step (public API) with each step's gradients H2D from pinned host memory and all "
                       "parameters D2H; amortised over f like value"}
        del host_grads

    # ---- fused Adam on the same shapes
    adam_ms = None
    if not args.skip_adam:
        ap = [p.clone().requires_grad_(True) for p in params]
        for p_, g_ in zip(ap, fresh()):
            p_.grad = g_.clone()
        adam = torch.optim.Adam(ap, lr=1e-3, fused=True)
        for _ in range(3):
            adam.step()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(20):
            adam.step()
        a1.record(stream)
        torch.cuda.synchronize()
        adam_ms = a0.elapsed_time(a1) / 20
        del ap, adam

    # the paper's per-iteration overhead: (Shampoo - Adam) / (fwd+bwd + Adam), with a
    # ResNet-50 fwd+bwd at batch 128 per GPU (bf16 autocast, channels_last, synthetic images)
    overhead = None
    if not args.skip_adam and rank == 0 and args.workload == "resnet50":
        try:
            import torchvision
            net = torchvision.models.resnet50().to(dev).to(memory_format=torch.channels_last)
            x = torch.randn(128, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
            y = torch.randint(0, 1000, (128,), device=dev)
            lossf = torch.nn.CrossEntropyLoss()

            def fwd_bwd():
                with torch.autocast("cuda", dtype=torch.bfloat16):
                    loss = lossf(net(x), y)
                loss.backward()

            for _ in range(3):
                fwd_bwd()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(10):
                fwd_bwd()
            f1.record()
            torch.cuda.synchronize()
            fb_ms = f0.elapsed_time(f1) / 10
            overhead = {"fwd_bwd_ms": round(fb_ms, 3), "batch_per_gpu": 128, "dtype": "bf16 autocast",
                        "overhead_vs_adam": round((value - adam_ms) / (fb_ms + adam_ms), 4),
                        "shampoo_over_adam": round(value / adam_ms, 2),
                        "paper": "6.70% at b=2048 f=50 on 8x V100 (PAPER.md:1245)",
                        "note": "(amortised Shampoo step - fused Adam step) / (fwd+bwd + Adam step); with J ranks "
                                "each rank preconditions ~1/J of the blocks"}
            del net, x, y
        except Exception as exc:  # torchvision missing or OOM: the optimizer numbers stand on their own
            overhead = {"unavailable": str(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu and args.workload in ("resnet50", "mlp"):
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
        r = cpu_reference(args.workload, 1)
        cpu = {"value": round(r["amortized_ms"], 2), "unit": "ms", "cores": r["cores"], "kind": "port",
               "sample": r["sample"], "plain_ms": round(r["plain_ms"], 1),
               "refresh_ms": round(r["refresh_extra_ms"], 1)}

    if rank == 0:
        nb = len(opt._blocks)
        line = {"metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 4),
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64" if args.precision == "double" else "f32", "data": "synthetic",
                "config": {"workload": f"{args.workload}_shampoo_step", "params": n_params, "blocks": nb,
                           "max_preconditioner_dim": wl["max_preconditioner_dim"], "precondition_frequency": f,
                           "grafting": wl["grafting"], "momentum": "nesterov 0.9", "precision": args.precision,
                           "epsilon": 1e-12, "parallelism": f"dp{world} (block-sharded, all-gather)",
                           "steady_state_from_step": T0, "check_finite": args.check_finite, "fast_forward_s": round(ff_s, 1),
                           "amortisation": "value = ((f-1) * mean(plain steps) + mean(refresh steps)) / f over the "
                                           "timed window, which starts at a steady-state refresh step",
                           "l2": "state (factors+inverses ~2 GB) >> 126 MB L2; no flush needed",
                           "gradients": "fresh N(0, 0.01^2) fp32 per step, resident in HBM (distinct "
                                        "within each window up to 8 GB of sets)"},
                "window_ms_per_step": round(window_ms, 4),
                "plain_step_ms": round(plain_ms, 4) if plain_ms else None,
                "refresh_step_ms": round(refresh_ms, 3) if refresh_ms else None,
                "refresh_steps_in_window": int(sum(refr)),
                "root_inverse_ms_per_block": round(per_call["root_inverse"] / max(nb, 1), 4),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "host_ms_per_step": round(1e3 * host_s / args.steps, 3),
                "host_enqueue_ms_per_plain_step": round(host_enqueue_ms, 3) if host_enqueue_ms is not None else None,
                "clocks": clk.summary(), "adam_fused_ms": round(adam_ms, 4) if adam_ms else None,
                "iteration_overhead": overhead,
                "device_state_gb": round(opt.device_bytes / 1e9, 3)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- config 5: root-inverse sweep


def run_sweep(args):
    """BASELINE config 5: batched eigh vs coupled-Newton root inverse on SPD factors Q diag(lam) Q^T,
    lam log-spaced over cond 1e6 (oracles.py:448-454 pattern), d in 128..8192, p in {2, 4}.
    Per (d, p, solver): device ms per block (CUDA events, best of reps), parity vs the float64
    CPU eigh oracle at every size, and the CPU oracle's ms beside it (sizes <= cpu_max)."""
    import torch

    import paper_2309_06497_b200 as P
    from oracle import shampoo_oracle as O

    dev = torch.device("cuda:0")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    sizes = [int(x) for x in args.sizes.split(",")]
    rng = np.random.default_rng(0)
    for d in sizes:
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        lam = np.exp(np.linspace(0.0, np.log(1e6), d)) * 1e-6
        a = (q * lam) @ q.T
        a = (a + a.T) / 2
        at = torch.as_tensor(a, device=dev)
        batch = max(1, args.sweep_batch if d <= 1024 else 1)
        mats = [at] * batch
        for p in (2, 4):
            ref = None
            cpu_ms = None
            if d <= args.cpu_max:
                t0 = time.perf_counter()
                ref = O.root_inverse_eigh(a, p, eps=1e-12)
                cpu_ms = 1e3 * (time.perf_counter() - t0)
            else:
                w, v = np.linalg.eigh(a)  # parity reference only (not timed)
                ref = (v * np.maximum(w - min(w.min(), 0) + 1e-12, 0) ** (-1.0 / p)) @ v.T
            for solver in ("eigh", "newton"):
                outs, status, its = P.batched_root_inverse(mats, p, epsilon=1e-12, solver=solver)
                torch.cuda.synchronize()
                best = 1e30
                for _ in range(args.sweep_reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    outs, status, its = P.batched_root_inverse(mats, p, epsilon=1e-12, solver=solver)
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                x = outs[0].cpu().numpy()
                err = float(np.linalg.norm(x - ref) / np.linalg.norm(ref))
                print(json.dumps({"sweep": "rootinv", "d": d, "p": p, "solver": solver, "batch": batch,
                                  "ms_per_block": round(best / batch, 3), "status": status[0],
                                  "iterations": its[0], "rel_err_vs_oracle": err,
                                  "cpu_oracle_ms": round(cpu_ms, 1) if cpu_ms else None,
                                  "cond": 1e6, "epsilon": 1e-12}), flush=True)


# ---------------------------------------------------------------- launcher


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["double", "single"], default="double")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="resnet50")
    ap.add_argument("--steady-step", type=int, default=-1,
                    help="first timed step (a refresh); -1: ceil(1.25 b / f) f (2600 for ResNet-50); 0: right "
                         "after the warm-up")
    ap.add_argument("--check-finite", choices=["deferred", "strict"], default="deferred",
                    help="non-finite gradient guard: device-predicated, raised one call late (no host sync), "
                         "or the reference's eager raise (one host sync per step)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-adam", action="store_true")
    ap.add_argument("--sweep", choices=["rootinv"], default=None)
    ap.add_argument("--sizes", default="128,256,512,1024,2048,4096,8192")
    ap.add_argument("--sweep-batch", type=int, default=4)
    ap.add_argument("--sweep-reps", type=int, default=2)
    ap.add_argument("--cpu-max", type=int, default=4096)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.sweep:
        run_sweep(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU under torchrun (the driver launches it that way itself)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
