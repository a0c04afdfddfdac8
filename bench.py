#!/usr/bin/env python
"""bench.py -- GDoF/s per FP64 operator apply on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 5, the largest single-GPU config:
alpha curl curl + beta (N1) on the 2x2x2 Kuhn cube mesh (48 macro-tets),
L = 8, 941,884,928 edge DoFs, weak-scaled with N (48 macros per GPU:
N=2 2x2x4, N=4 2x4x4, N=8 4x4x4 = 384 macros). The other configs
(c1..c4) run with --config; c4 (P1 -Laplace, cube6 L8) is strong-scaled.

A "step" = one operator apply y = A x (element kernel + interface sum +
cross-rank exchange) over the whole mesh, inputs resident in HBM. Inputs of
every config exceed L2 except c1-c3 (latency-bound parity configs), which
flush L2 between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
  python bench.py --impl reference ...   # the reference's CPU apply

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
torch.cuda.synchronize(), CUDA events on the stream the kernels run on, max
over ranks. e2e: the same metric through the public C-ABI drop-in
(tetmf_apply_ref_host: host vectors in reference numbering, H2D + apply +
D2H every step, pinned buffers) at N=1; per-rank upload/apply/download of
the local storage for N>1.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDoF/s per operator apply (FP64) at 1/2/4/8 B200; fraction of roofline"

# F = flop per element of the cheapest exact formulation counted with
# DFMA = 2; M = compulsory bytes per DoF.
CONFIGS = {
    "c1": dict(name="P1 -Laplace single-tet L6 (config 1)", mesh="single-tet", form="P1", level=6, dirichlet=True),
    "c2": dict(name="P1 -div(k grad) single-tet L7 (config 2)", mesh="single-tet", form="P1K", level=7),
    "c3": dict(name="N1 alpha curl curl + beta single-tet L6 (config 3)", mesh="single-tet", form="N1", level=6),
    "c4": dict(name="P1 -Laplace cube6 L8 (config 4, strong scaling)", mesh="cube6", form="P1", level=8),
    "c5": dict(name="N1 alpha curl curl + beta, 48 macros/GPU L8 (config 5, weak scaling)", mesh=None,
               form="N1", level=8),
    # config 2's form (P1 -div(k grad)) at config 4's bandwidth-bound size
    "c2l": dict(name="P1 -div(k grad) cube6 L8 (config 2's form at config 4's size)", mesh="cube6", form="P1K",
                level=8),
    # SURVEY.md 8(f) #2 (not a BASELINE config): the paper's P2V form
    "p2v": dict(name="P2V -div(k grad), u and k in P2, cube6 L8 (SURVEY 8(f) #2)", mesh="cube6", form="P2V",
                level=8),
}
WEAK_MESH = {1: "cubes2x2x2", 2: "cubes2x2x4", 4: "cubes2x4x4", 8: "cubes4x4x4"}
CPU_SAMPLE = {  # bounded sample of each workload for the CPU reference leg
    "c1": ("single-tet", 6), "c2": ("single-tet", 6), "c3": ("single-tet", 5),
    "c4": ("cube6", 6), "c5": ("cubes2x2x2", 4), "p2v": ("cube6", 4), "c2l": ("cube6", 6),
}
# P2V: the factored algorithm's count (k_p2v.cu: K 190, U 28, W 112, Z 112,
# contractions 28, accumulation 10 flop); the table form needs 1300
FLOP_PER_ELEM = {"P1": None, "P1K": None, "N1": 264.0, "P2V": 480.0}


def lattice_counts(mesh_macros: int, level: int, form: str):
    n = 1 << level
    tet = lambda k: (k + 1) * (k + 2) * (k + 3) // 6 if k >= 0 else 0
    return dict(elements=mesh_macros * n ** 3, p1_points=mesh_macros * tet(n),
                nd1_edges=mesh_macros * (6 * tet(n - 1) + tet(n - 2)))


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": reasons, "samples": len(self.samples)}
        if getattr(self, "window", None):
            out["window"] = self.window
        return out


# ------------------------------------------------------------------ CPU legs
def cpu_reference_sample(cfg_key: str, seconds: float = 12.0, verbatim: bool = True):
    """Times the reference's own FormSystem::apply (oracle/_ref, compiled from
    the reference sources) single-threaded on a bounded sample of the
    workload. Returns (GDoF/s, sample description, dofs, seconds/apply)."""
    import tempfile

    from oracle.refapi import RefSystem, write_kuhn_mesh
    cfg = CONFIGS[cfg_key]
    mesh, level = CPU_SAMPLE[cfg_key]
    mesh_arg = mesh
    if mesh.startswith("cubes"):  # the reference loads K^3 Kuhn meshes from its text format
        k = [int(v) for v in mesh[5:].split("x")]
        k = k * 3 if len(k) == 1 else k
        mesh_arg = os.path.join(tempfile.gettempdir(), f"tetmf_{mesh}.mesh")
        write_kuhn_mesh(mesh_arg, *k)
    r = RefSystem(mesh_arg, cfg["form"], level, fixed=not verbatim)
    x = r.seeded_input(42)
    c0, c1 = r.coefficients()
    # same rule class as the GPU: exact, cheapest (P1: 2, N1: 3, P2V: 4)
    degree = {"N1": 3, "P2V": 4}.get(cfg["form"], 2)
    r.apply(x, c0, c1, degree)  # warm-up fills the star / map caches
    times = []
    t_end = time.time() + seconds
    while time.time() < t_end or len(times) < 3:
        _, t = r.apply(x, c0, c1, degree)
        times.append(t)
    t = float(np.median(times))
    return r.num_dofs / t / 1e9, f"{mesh} L{level} {cfg['form']} ({r.num_dofs} DoFs, degree-{degree} rule, " \
                                 f"median of {len(times)} applies)", r.num_dofs, t


def _replica(args):
    cfg_key, seconds = args
    g, _, dofs, t = cpu_reference_sample(cfg_key, seconds)
    return dofs, t


def run_reference_arm(a):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[a.config]
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        pass
    mesh, level = CPU_SAMPLE[a.config]
    # the reference is single-threaded and not thread-safe (mutable caches,
    # forms.hpp:86-87): one replica process per host core, aggregate DoF/s
    nrep = max(1, min(cores, int(os.environ.get("TETMF_REF_REPLICAS", "64"))))
    per_step = []
    with mp.get_context("fork").Pool(nrep) as pool:
        for _ in range(a.warmup):
            pool.map(_replica, [(a.config, 0.0)] * nrep)
        for _ in range(a.steps):
            t0 = time.time()
            res = pool.map(_replica, [(a.config, 0.0)] * nrep)
            per_step.append(sum(d for d, _ in res) / max(t for _, t in res) / 1e9)
    v = float(np.median(per_step))
    sample = f"{nrep} concurrent single-thread replicas of the verbatim reference FormSystem::apply on " \
             f"{mesh} L{level} {cfg['form']}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GDoF/s", "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak" if a.config == "c5" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1] x, nodal coefficients)",
        "config": {"workload": cfg["name"], "cpu_sample": f"{mesh} L{level}", "level": cfg["level"]},
        "cpu_baseline": {"value": v, "unit": "GDoF/s", "cores": nrep, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ GPU leg
def roofline(cfg_key, form, local_counts, kern_avg_ms, ms_per_step, fp64_peak):
    """Roofline of the dominant (element) kernel: algorithmic flops (N1, P2V:
    FLOP_PER_ELEM x elements) or compulsory bytes (P1: x + y, P1K: x + k + y
    per point) per launch / its CUDA-event duration, against the measured
    peak; traffic = ncu DRAM bytes per launch from the committed capture."""
    traffic = None
    for name in ("r2_traffic.json", "r1_traffic.json"):
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", name))).get(cfg_key)
        except Exception:
            traffic = None
        if traffic:
            break
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sec = kern_avg_ms * 1e-3
    if form in ("N1", "P2V"):
        nd1_local, p1_local = local_counts["nd1_edges"], local_counts["p1_points"]
        # F = the cheapest exact formulation's flops, and the
        # builder's ncu-measured FP64 flop count replaces it when lower
        # (profiles/r2_flops.json: executed DFMA x 2 + DADD + DMUL per element)
        f_survey = FLOP_PER_ELEM[form]
        meas = None
        try:
            meas = json.load(open(os.path.join(ROOT, "profiles", "r2_flops.json"))).get(form)
        except Exception:
            meas = None
        f_eff = min(f_survey, meas["flop_per_element"]) if meas else f_survey
        flops = f_eff * local_counts["elements"]
        # N1: x, y (edges) + alpha, beta (points); P2V: x, k, y (points + edges)
        bytes_alg = 8.0 * ((2 * nd1_local + 2 * p1_local) if form == "N1" else 3 * (nd1_local + p1_local))
        roof = {"bound": "fp64", "achieved": flops / sec / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": (flops / sec / 1e12) / fp64_peak if fp64_peak else None,
                "flop_per_launch": flops, "flop_per_element": f_eff,
                "flop_per_element_survey": f_survey,
                "frac_at_survey_F": (f_survey * local_counts["elements"] / sec / 1e12) / fp64_peak if fp64_peak else None,
                "flop_per_element_measured": meas["flop_per_element"] if meas else None,
                "flop_measured_source": meas["source"] if meas else None,
                "peak_source": "measured FP64 DFMA-chain probe on this GPU: best launch of a 4 s window "
                               "(tetmf_measure_fp64_peak2; peak_sustained = its second half)",
                "hbm": {"achieved": bytes_alg / sec / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "bytes_per_launch": bytes_alg}}
    else:
        nbytes = 8.0 * local_counts["p1_points"] * (3 if form == "P1K" else 2)
        roof = {"bound": "hbm", "achieved": nbytes / sec / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "frac": nbytes / sec / 1e9 / hbm_peak, "bytes_per_launch": nbytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    roof["traffic"] = traffic["bytes_per_launch"] if traffic else None
    roof["traffic_source"] = traffic["source"] if traffic else None
    roof["kernel_ms"] = kern_avg_ms
    roof["kernel_share_of_step"] = kern_avg_ms / ms_per_step
    return roof


def make_operator(tm, ctx, form, level, dirichlet=False, seed=42):
    fid = {"P1": tm.FORM_P1, "P1K": tm.FORM_P1K, "N1": tm.FORM_N1, "P2V": tm.FORM_P2V}[form]
    sid = tm.FORM_SPACE[fid]
    x, y = tm.Function(ctx, sid), tm.Function(ctx, sid)
    coeffs = []
    if form == "N1":
        al, be = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        al.fill_coefficient(level, tm.COEFF_ALPHA)
        be.fill_coefficient(level, tm.COEFF_BETA)
        coeffs = [al, be]
    elif form in ("P1K", "P2V"):
        k = tm.Function(ctx, tm.SPACE_P1 if form == "P1K" else tm.SPACE_P2)
        k.fill_coefficient(level, tm.COEFF_K)
        coeffs = [k]
    op = tm.Operator(ctx, fid, coeffs)
    x.fill_seeded(level, seed, dirichlet)
    y.size(level)
    return op, x, y, coeffs


def sub_record(tm, torch, key, steps, warmup, device, fp64_peak):
    """One single-GPU config timed like the headline (events on the context
    stream, kernel events, L2 flushed between steps when the inputs fit in
    it), returned as a sub-record of the default bench line so that the
    driver's record carries every operator's roofline, not only config 5's."""
    cfg = CONFIGS[key]
    level, form = cfg["level"], cfg["form"]
    ctx = tm.Context(cfg["mesh"], device=device)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    op, x, y, _ = make_operator(tm, ctx, form, level, cfg.get("dirichlet", False))
    nmac = ctx.num_macros()[0]
    counts = lattice_counts(nmac, level, form)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") \
        if counts["elements"] < 50_000_000 else None
    for _ in range(warmup):
        op.apply(x, y, level)
    torch.cuda.synchronize()
    # Pass 1 (the value): no events between the kernels of an apply. Events
    # there cost ~8 us per apply at config 4 and keep the kernels' programmatic
    # dependent launches (K1 / K4, runtime_check.hpp) from overlapping. Inputs
    # larger than L2: the steps run back to back inside one event bracket, as a
    # solver issues them. Inputs that fit: one bracket per step, L2 flushed
    # outside it.
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            op.apply(x, y, level)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    else:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            flush.zero_()
            ev[i][0].record(stream)
            op.apply(x, y, level)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(s.elapsed_time(e) for s, e in ev) / steps
    # Pass 2 (the roofline's kernel time): the same steps with the library's
    # events around the element kernel of every apply
    op.profile(True)
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        op.apply(x, y, level)
    torch.cuda.synchronize()
    kern_ms, kern_n = op.kernel_stats()
    op.profile(False)
    n_unique = unique_dofs(cfg["mesh"], form, level)
    rec = {"workload": cfg["name"], "mesh": cfg["mesh"], "level": level, "form": form, "dofs": n_unique,
           "value": n_unique / (ms * 1e-3) / 1e9, "unit": "GDoF/s", "ms_per_step": ms, "steps": steps,
           "l2": "inputs > 126 MB L2" if flush is None else "L2 flushed between steps",
           "timing": ("one CUDA-event bracket around the steps, applies back to back" if flush is None else
                      "one CUDA-event bracket per step") + "; kernel_ms from a second pass of the same steps with "
                     "events around the element kernel",
           "roofline": roofline(key, form, lattice_counts(nmac, level, form), kern_ms / max(kern_n, 1), ms,
                                fp64_peak)}
    del op, x, y, ctx
    torch.cuda.synchronize()
    return rec


def run_gpu(a):
    import torch
    import torch.distributed as dist

    import paper_2404_08371_b200 as tm

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    # one explicit (non-default) stream for torch's events / flushes and the
    # library's kernels: tetmf_ctx_set_stream(NULL) would select the
    # context's own stream, and torch's default stream handle is NULL
    torch.cuda.set_stream(torch.cuda.Stream())
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = dict(CONFIGS[a.config])
    if cfg["mesh"] is None:
        if ws not in WEAK_MESH:
            raise SystemExit(f"config c5 supports 1/2/4/8 GPUs, got {ws}")
        cfg["mesh"] = WEAK_MESH[ws]
    level, form = cfg["level"], cfg["form"]
    fid = {"P1": tm.FORM_P1, "P1K": tm.FORM_P1K, "N1": tm.FORM_N1, "P2V": tm.FORM_P2V}[form]
    sid = tm.FORM_SPACE[fid]

    nccl_id = None
    if ws > 1:
        obj = [tm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t_setup = time.time()
    # config 4 (strong scaling, 6 macros): (macro, z-slab) units over the ranks
    slab = a.config == "c4" and ws > 1
    ctx = tm.Context(cfg["mesh"], device=local, rank=rank, nranks=ws, nccl_id=nccl_id,
                     partition=tm.PARTITION_SLAB if slab else tm.PARTITION_MACRO)
    if ws > 1 and a.exchange == "put":
        ctx.set_exchange_mode(tm.EXCHANGE_PUT)  # before the first level: the put channel opens with it
    comm_info = ctx.transport_info()  # "nccl rank r of N (cuda device d)": the communicator's own rank count
    if ws > 1:
        comm_info += f"; interface exchange: {a.exchange}"
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    nmac_global, nmac_local = ctx.num_macros()
    x, y = tm.Function(ctx, sid), tm.Function(ctx, sid)
    coeffs = []
    if form == "N1":
        al, be = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        al.fill_coefficient(level, tm.COEFF_ALPHA)
        be.fill_coefficient(level, tm.COEFF_BETA)
        coeffs = [al, be]
    elif form in ("P1K", "P2V"):
        k = tm.Function(ctx, tm.SPACE_P1 if form == "P1K" else tm.SPACE_P2)
        k.fill_coefficient(level, tm.COEFF_K)
        coeffs = [k]
    op = tm.Operator(ctx, fid, coeffs)
    if a.variant:
        op.set_variant(a.variant)  # kernel A/B (0 = default optimized kernels)
    x.fill_seeded(level, 42, cfg.get("dirichlet", False))
    y.size(level)
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup

    counts = lattice_counts(nmac_global, level, form)
    n_unique = None
    # unique DoFs of the whole mesh (reference numbering count)
    if rank == 0 and ws == 1:
        n_unique = x.num_ref_dofs(level)
    if n_unique is None:
        n_unique = unique_dofs(cfg["mesh"], form, level)

    small = counts["elements"] < 50_000_000
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if small else None

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(a.warmup):
        if flush is not None:
            flush.zero_()
        op.apply(x, y, level)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with ClockSampler(local) as clk:
        # nvidia-smi samples every 100 ms; when the timed region is shorter,
        # untimed applies keep the GPU under the same load until the sampler
        # has seen it (before) and once more after the timed steps, so the
        # samples bracket the timed region (clk.window says which)
        def load_until(count, limit_s=3.0):
            t_end = time.time() + limit_s
            while len(clk.samples) < count and time.time() < t_end:
                for _ in range(4):
                    op.apply(x, y, level)
                torch.cuda.synchronize()
        load_until(2)
        n_before = len(clk.samples)
        lc0 = tm.launch_count()
        op.profile(True)
        for i in range(a.steps):
            if flush is not None:
                flush.zero_()  # L2 flush outside the timed interval of each step
            ev[i][0].record(stream)
            op.apply(x, y, level)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        launches = tm.launch_count() - lc0
        kern_ms, kern_n = op.kernel_stats()
        op.profile(False)
        n_during = len(clk.samples) - n_before
        load_until(len(clk.samples) + 1)
        clk.window = ("timed region" if n_during >= 2 else
                      f"untimed applies under the same load immediately before / after the timed region "
                      f"({n_during} sample(s) inside it)")
    barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    t_total = sum(step_ms)
    if ws > 1:
        tt = torch.tensor([t_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    ms_per_step = t_total / a.steps
    value = n_unique / (ms_per_step * 1e-3) / 1e9

    # ---------------- roofline of the dominant (element) kernel
    kern_avg_ms = kern_ms / max(kern_n, 1)
    fp64_peak = fp64_sustained = None
    if a.fp64_peak and form in ("N1", "P2V"):
        fp64_peak, fp64_sustained = ctx.fp64_peak2(4.0)
    local_counts = lattice_counts(nmac_local, level, form)
    if slab:  # this rank's points: its units' planes
        n = 1 << level
        local_counts["p1_points"] = sum((n + 1 - z) * (n + 2 - z) // 2 for _, za, zb in
                                        tm.slab_units(nmac_global, level, ws, rank) for z in range(za, zb))
    roof = roofline(a.config, form, local_counts, kern_avg_ms, ms_per_step, fp64_peak)
    if fp64_sustained:  # the probe's rate once the clocks settle (reported beside the burst-peak frac)
        roof["peak_sustained"] = fp64_sustained
        roof["frac_vs_sustained"] = roof["achieved"] / fp64_sustained

    # ---------------- end to end through the public API (host buffers)
    e2e = None
    if a.e2e:
        e2e = run_e2e(a, tm, torch, dist, ctx, op, x, y, level, ws, rank, n_unique, barrier)

    # the other operators' rooflines at their bandwidth-bound sizes (1 GPU)
    subs = {}
    if a.subrecords and ws == 1 and a.config == "c5":
        del x, y
        for key in ("c4", "c2l", "p2v", "c1", "c2", "c3"):
            subs[key] = sub_record(tm, torch, key, max(a.steps, 10), 3, local, fp64_peak)

    cpu = None
    if rank == 0 and ws == 1 and a.cpu_baseline:
        try:
            g, sample, _, _ = cpu_reference_sample(a.config, seconds=a.cpu_seconds)
            cpu = {"value": g, "unit": "GDoF/s", "cores": 1, "kind": "reference",
                   "sample": "verbatim reference FormSystem::apply (oracle/_ref, -O3), 1 host core, " + sample}
        except Exception as e:  # the reference lib is built here and ships with the snapshot
            cpu = {"value": None, "unit": "GDoF/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if a.config == "c5" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: x seeded uniform[-1,1] by canonical DoF key (SURVEY 8(d)); nodal coefficients (P1; P2 for P2V)",
            "config": {"workload": cfg["name"], "mesh": cfg["mesh"], "level": level, "form": form,
                       "macros": nmac_global, "dofs": n_unique, "elements": counts["elements"],
                       "parallelism": (f"(macro, z-slab) partition over {ws} GPU(s)" if slab else
                                       f"macro partition over {ws} GPU(s)"), "comm": comm_info,
                       "l2": "inputs > 126 MB L2" if flush is None else "L2 flushed between steps",
           "timing": ("one CUDA-event bracket around the steps, applies back to back" if flush is None else
                      "one CUDA-event bracket per step") + "; kernel_ms from a second pass of the same steps with "
                     "events around the element kernel",
                       "setup_s": round(t_setup, 2)},
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if subs:
            out["subrecords"] = subs
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def unique_dofs(mesh: str, form: str, level: int) -> int:
    """Unique DoFs of a Kuhn cube mesh / built-in mesh (closed forms,
    SURVEY.md Appendix B): P1 (N+1)^3 vertices; ND1 7N^3 + 9N^2 + 3N edges."""
    import re
    if form == "P2V":  # P2: vertices + edge midpoints
        return unique_dofs(mesh, "P1", level) + unique_dofs(mesh, "N1", level)
    n = 1 << level
    if mesh == "single-tet":
        tet = lambda k: (k + 1) * (k + 2) * (k + 3) // 6
        return tet(n) if form != "N1" else 6 * tet(n - 1) + tet(n - 2)
    m = re.fullmatch(r"cubes(\d+)x(\d+)x(\d+)", mesh) or re.fullmatch(r"cubes(\d+)", mesh)
    k = [int(g) for g in m.groups()] if m else [1, 1, 1]
    if len(k) == 1:
        k = k * 3
    N = [ki * n for ki in k]
    if form != "N1":
        return (N[0] + 1) * (N[1] + 1) * (N[2] + 1)
    X, Y, Z = N
    # edges: axis (3), face diagonals (3), body diagonal (1) of every cube
    axis = X * (Y + 1) * (Z + 1) + (X + 1) * Y * (Z + 1) + (X + 1) * (Y + 1) * Z
    faces = X * Y * (Z + 1) + X * (Y + 1) * Z + (X + 1) * Y * Z
    return axis + faces + X * Y * Z


def pcie_duplex_gbs(torch, nbytes=1 << 30, reps=3):
    """GB/s per direction of concurrent pinned H2D + D2H copies (the e2e bound)."""
    n = nbytes // 8
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float64, device="cuda")
    d_out = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    both()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        both()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / reps
    del h_in, h_out, d_in, d_out
    return n * 8 / sec / 1e9


def run_e2e(a, tm, torch, dist, ctx, op, x, y, level, ws, rank, n_unique, barrier):
    steps = max(1, min(a.steps, a.e2e_steps))
    if ws == 1:
        nd = x.num_ref_dofs(level)
        hv = tm.host_alloc(nd * 8)
        hw = tm.host_alloc(nd * 8)
        try:
            # host input vector in reference numbering (the FieldVector a caller holds)
            x.export_ref(level)  # builds the numbering maps (setup, untimed)
            arr = np.ctypeslib.as_array((ctypes_double_p(hv)), shape=(nd,))
            arr[:] = x.export_ref(level)
            src, dst = tm.Function(ctx, x.space), tm.Function(ctx, x.space)
            op.apply_ref_host(src, dst, level, hv, hw)  # warm-up
            t = []
            for _ in range(min(steps, 3)):  # the synchronous call, reported beside the batch
                t0 = time.perf_counter()
                op.apply_ref_host(src, dst, level, hv, hw)
                t.append(time.perf_counter() - t0)
            sec1 = float(np.median(t))
            # the batched drop-in: `steps` applies in ONE C-ABI call, each with
            # its own H2D of the input and D2H of its result, pipelined over
            # three streams (copy-in k+1 || permute/apply/permute k || copy-out k-1)
            op.apply_ref_host_batch(src, dst, level, [hv] * 2, [hw] * 2)  # warm-up
            t0 = time.perf_counter()
            op.apply_ref_host_batch(src, dst, level, [hv] * steps, [hw] * steps)
            sec = (time.perf_counter() - t0) / steps
            pcie = pcie_duplex_gbs(torch)
            return {"value": n_unique / sec / 1e9, "unit": "GDoF/s", "h2d_bytes_per_step": nd * 8,
                    "d2h_bytes_per_step": nd * 8, "ms_per_step": sec * 1e3, "steps": steps,
                    # the e2e step moves nd doubles each way: its bound is the
                    # concurrent H2D + D2H bandwidth of this box's PCIe link
                    "roofline": {"bound": "pcie", "achieved": nd * 8 / sec / 1e9, "peak": pcie, "unit": "GB/s per direction",
                                 "frac": nd * 8 / sec / 1e9 / pcie,
                                 "peak_source": "measured here: concurrent pinned H2D + D2H copies of 1 GiB (torch)"},
                    "path": "tetmf_apply_ref_host_batch (one call, `steps` applies): pinned host FieldVector "
                            "(reference numbering) -> H2D -> permute -> apply -> permute -> D2H per apply, copies "
                            "pipelined over three streams",
                    "single_call": {"value": n_unique / sec1 / 1e9, "ms_per_step": sec1 * 1e3,
                                    "path": "tetmf_apply_ref_host per apply (synchronous)"}}
        finally:
            tm.host_free(hv)
            tm.host_free(hw)
    # N > 1: each rank holds its owned slice of the global FieldVector in
    # reference numbering (pinned): H2D + ghost update + apply + D2H of the
    # owned slice (tetmf_fn_import_ref_owned / export_ref_owned)
    lo, hi = x.owned_ref_range(level)
    nown = hi - lo
    hv = tm.host_alloc(max(nown, 1) * 8)
    hw = tm.host_alloc(max(nown, 1) * 8)
    try:
        np.ctypeslib.as_array(ctypes_double_p(hv), shape=(max(nown, 1),))[:] = 0.5
        src, dst = tm.Function(ctx, x.space), tm.Function(ctx, x.space)
        src.import_ref_owned(level, hv)  # warm-up (collective)
        op.apply(src, dst, level)
        dst.export_ref_owned(level, hw)
        t = []
        for _ in range(steps):
            barrier()
            t0 = time.perf_counter()
            src.import_ref_owned(level, hv)
            op.apply(src, dst, level)
            dst.export_ref_owned(level, hw)
            t.append(time.perf_counter() - t0)
    finally:
        tm.host_free(hv)
        tm.host_free(hw)
    tt = torch.tensor([float(np.median(t))], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    sec = float(tt.item())
    return {"value": n_unique / sec / 1e9, "unit": "GDoF/s", "h2d_bytes_per_step": nown * 8,
            "d2h_bytes_per_step": nown * 8, "ms_per_step": sec * 1e3, "steps": steps,
            "path": "per rank: owned slice of the FieldVector (reference numbering, pinned) -> H2D -> "
                    "tetmf_fn_import_ref_owned (ghost copies from their owners over the transport) -> apply -> "
                    "tetmf_fn_export_ref_owned -> D2H (synchronous per step; max over ranks)"}


def ctypes_double_p(addr):
    import ctypes
    return ctypes.cast(ctypes.c_void_p(addr), ctypes.POINTER(ctypes.c_double))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    p.add_argument("--no-e2e", dest="e2e", action="store_false")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-fp64-peak", dest="fp64_peak", action="store_false")
    p.add_argument("--variant", type=int, default=0, help="kernel variant for A/B runs (0 = default)")
    p.add_argument("--exchange", choices=["sendrecv", "put"], default="sendrecv",
                   help="N > 1: interface exchange by NCCL send/recv or by direct NVLink puts (NCCL device API)")
    p.add_argument("--no-subrecords", dest="subrecords", action="store_false",
                   help="c5 only: skip the c4 / c2l / p2v / c1-c3 sub-records")
    a = p.parse_args()
    a.warmup = max(a.warmup, 3)
    if a.impl == "reference":
        run_reference_arm(a)
        return
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and a.gpus > 1:
        sys.exit(launch_ranks(a))
    if ws and ws != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={ws}")
    run_gpu(a)


def launch_ranks(a) -> int:
    """--gpus N without a launcher: re-exec this script under torchrun, one
    rank per GPU (127.0.0.1 rendezvous). Fails loudly when fewer than N GPUs
    are visible -- N ranks never share a device in the bench."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"error": f"--gpus {a.gpus} requested but only {have} CUDA device(s) visible"}),
              file=sys.stderr, flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
