"""Benchmark of the plain rank-1 lattice sum (BASELINE.json metric: lattice
f-evals/s in FP64, % of FP64 peak; MDI-LR time-to-solution reported beside).

Workload (``config.workload``): BASELINE config 5's plain sum -- d=1000,
prime n=2^31-1, seeded Korobov z, f(x)=exp(-|sum c_j (x_j - w_j)|) -- the
largest single-GPU configuration and the only one big enough to measure the
FP64 roofline (configs 1-3 take <=0.2 ms; they are parity cases).
One step = one full sum over all n points.  Multi-GPU: super-chunks of the
index range are split across ranks, the per-super-chunk partials meet in one
NCCL all-reduce (disjoint slots, so exact) and a fixed-order tree -- results
are bit-identical for any GPU count.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "lattice f-evals/sec (fp64) & MDI-LR time-to-solution; % of FP64 peak"   # BASELINE.json
FLOPS_PER_PD = 3          # 1 (coordinate r/n) + 2 (c_j * x_j accumulate) for exp-abs-linear
FLOPS_PER_POINT = 2       # transcendental + accumulate
TERM_FLOPS = 2            # SURVEY.md §8(d) per-coordinate term of exp-abs-linear (c_j * x_j accumulate)
ORB_M = 24                # points per chain of the orbit kernel (LQ_ORB_LIN_M, csrc/lq_kernels.cu)
FFT_N = 4096              # transform length of the FFT-form orbit kernel (kFftN, csrc/lq_fft.cuh)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, power = [], [], set(), []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                mask = int(parts[2], 16)
                power.append(float(parts[3]) if len(parts) > 3 else float("nan"))
            except ValueError:
                continue
            for bit, name in REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": float(np.nanmax(power)) if power else None}


def cpu_model():
    """Host CPU model name (SURVEY §8d asks for it next to the CPU baseline)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_rate(npts, workers):
    """(pts/s, seconds, kind, what) of config 5's plain sum over its first
    ``npts`` points on the host: the reference itself from baseline/_ref
    (its lattice.points_block + the integrand in numpy) when installed, else
    the oracle's numpy restatement of the same (oracle/cpu_baseline.py)."""
    sys.path.insert(0, os.path.join(REPO, "baseline"))
    import ref_cpu
    t0 = time.perf_counter()
    if ref_cpu.available():
        ref_cpu.cfg5_range_sum(0, npts, workers=workers)
        kind, what = "reference", ("latquad.lattice.points_block from baseline/_ref (the reference itself) "
                                   "+ exp(-|x c - c.w|) in numpy")
    else:
        from oracle import cpu_baseline as cb
        from paper_2404_08867_b200.configs import make_config
        cb.cfg5_range_sum(make_config(5), 0, npts, workers=workers)
        kind, what = "port", "numpy restatement of lattice.points_block + integrand (oracle/np_oracle.py)"
    dt = time.perf_counter() - t0
    return npts / dt, dt, kind, what


def _suite_job(which):
    sys.path.insert(0, os.path.join(REPO, "baseline"))
    import ref_cpu
    return ref_cpu.suite_one(which)


def reference_suite():
    """The reference's public API as is on configs 1-3 (slr_integrate) and 2, 1
    (mdi_lr), each on one host core (five processes side by side); None when
    baseline/_ref is not installed."""
    sys.path.insert(0, os.path.join(REPO, "baseline"))
    import ref_cpu
    if not ref_cpu.available():
        return None
    import multiprocessing as mp
    jobs = ["slr1", "slr2", "slr3", "mdi2", "mdi1"]
    with mp.get_context("spawn").Pool(len(jobs)) as pool:
        res = pool.map(_suite_job, jobs)
    out = {}
    for r in res:
        out.update(r)
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path for config 5 on all host
    cores -- latquad itself from baseline/_ref (points_block + the integrand in
    numpy; the grammar has no |.|), else the oracle's restatement."""
    if rank != 0:
        return
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    cores = os.cpu_count() or 1
    sample = args.ref_sample
    for _ in range(args.warmup):
        ref_rate(sample // 4, cores)
    t = 0.0
    for _ in range(args.steps):
        rate, dt, kind, what = ref_rate(sample, cores)
        t += dt
    value = args.steps * sample / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "f-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg5_plain_sum", "d": cfg.d, "n": cfg.plain_n, "a": cfg.plain_a,
                   "integrand": "exp(-|sum c_j (x_j - w_j)|)", "sample_points_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "f-evals/s", "cores": cores, "kind": kind,
                         "sample": f"first {sample} points of cfg5 per step, {what}, contiguous index ranges "
                                   f"over {cores} processes",
                         "cpu_model": cpu_model(), "host_cores": os.cpu_count()},
        "e2e": {"value": value, "unit": "f-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=1 << 21)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--no-mdi", action="store_true")
    ap.add_argument("--no-ref-suite", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # one process per GPU; LQ_DIST_BACKEND=gloo lets the multi-rank logic be
    # exercised with several ranks sharing one GPU (no kernel waits on another)
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    backend = os.environ.get("LQ_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)

    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    from paper_2404_08867_b200.configs import make_config
    from paper_2404_08867_b200.distributed import exchange_disjoint

    h = N.lib()
    ctx = N.ctx(dev)
    # a dedicated (non-default) stream shared by liblq and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    N.check(h.lq_ctx_set_stream(ctx, C.c_void_p(stream.cuda_stream)))

    # cold first call of the public API in this process: text -> estimate,
    # including lowering, the orbit plan (primality, ord(a), primitive root,
    # chain-start tables), their upload, the coefficient transform and the sum
    cfg = make_config(5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    cold_est = lq.slr_integrate(f, rule).value
    cold_ms = (time.perf_counter() - t0) * 1e3
    n, d = rule.n, rule.d
    z = rule.z_reduced_array()
    pi = engine.plain_integrand(f, d)
    assert pi.kind == "lin_expabs", pi.kind

    # FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry, so the
    # DFMA probe in liblq measures it on this GPU, in this run (sustained ~1 s).
    tf, ms = C.c_double(), C.c_float()
    N.check(h.lq_fp64_peak(ctx, 1, C.byref(tf), C.byref(ms)))
    iters = max(1, int(1000.0 / max(ms.value, 1e-3)))
    N.check(h.lq_fp64_peak(ctx, iters, C.byref(tf), C.byref(ms)))
    fp64_peak = tf.value

    lay = N.lattice_layout(pi.struct, n, z)
    n_super = lay.n_supers
    s_lo, s_hi = n_super * rank // world, n_super * (rank + 1) // world
    parts = torch.zeros(n_super, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")     # 256 MiB > 126 MB L2
    out = C.c_double()

    def step():
        N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), n, N.as_ptr(z), s_lo, s_hi,
                                      C.c_void_p(parts.data_ptr() + 8 * s_lo)))
        if world > 1:
            exchange_disjoint(parts)    # disjoint slots: exact, order-independent
        N.check(h.lq_reduce_sum(ctx, C.c_void_p(parts.data_ptr()), n_super, C.byref(out)))
        return out.value

    for _ in range(args.warmup):
        parts.zero_()
        step()
    torch.cuda.synchronize()

    N.check(h.lq_ctx_enable_timing(ctx, 1))
    total_ms, kern_ms, launches = 0.0, 0.0, 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)          # L2 flush between timed steps, outside the event window
            parts.zero_()
            ev0.record(stream)
            value_sum = step()
            ev1.record(stream)
            ev1.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            kms, nl = C.c_float(), C.c_int64()
            N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
            kern_ms += kms.value
            N.check(h.lq_ctx_enable_timing(ctx, 1))
            launches += int(nl.value)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = args.steps * n / (total_ms * 1e-3)
    estimate = value_sum / n

    prof = {}
    prof_path = os.path.join(REPO, "profiles", "ncu_summary.json")
    if os.path.exists(prof_path):
        with open(prof_path) as fh:
            prof = json.load(fh)
    # dominant kernel roofline over this rank's units.  Orbit layout: a unit is
    # a chain of ORB_M points whose linear forms are computed once and serve
    # the point and its mirror; index layout: a unit is a point.
    su = lay.tile_units * lay.super_tiles
    my_units = min(s_hi * su, lay.n_units) - s_lo * su
    avg_kern = kern_ms / args.steps
    if lay.mode == N.LAYOUT_ORBIT_FFT:
        B = FFT_N - d + 1                              # points per chain (overlap-save block)
        forms = my_units * B                           # linear forms (one per mirrored pair)
        fft_flops = 2 * 5 * FFT_N * int(math.log2(FFT_N)) + 6 * FFT_N   # fwd + inv complex FFT + spectrum product
        alg_flops = (my_units / 2) * fft_flops + forms * 2 * FLOPS_PER_POINT
        conv_flops = forms * (FLOPS_PER_PD * d + 2 * FLOPS_PER_POINT)
        # FP64 flops the kernel actually executes (twiddle products, exponent
        # arithmetic, polynomial): per tile from the committed ncu capture
        exec_flops = (my_units / 2) * prof.get("k_orbit_fft", {}).get("fp64_flop_executed_per_tile", 0.0)
        kernel_name = "k_orbit_fft<OUT_EXPABS> (liblq.so)"
        unit_txt = (f"unit = chain of {B} mirrored point pairs, two chains per {FFT_N}-point complex FFT tile; "
                    f"per tile 2 x 5 N log2 N (forward + inverse FFT) + 6 N (spectrum product) flop, "
                    f"+ 2 x {FLOPS_PER_POINT} per pair (two outer evaluations)")
    elif lay.mode == N.LAYOUT_ORBIT:
        forms = my_units * ORB_M                       # linear forms evaluated (one per mirrored pair)
        alg_flops = forms * (TERM_FLOPS * d + 2 * FLOPS_PER_POINT)
        conv_flops = forms * (FLOPS_PER_PD * d + 2 * FLOPS_PER_POINT)
        exec_flops = forms * 2 * (-(-d // ORB_M) * ORB_M)   # DFMAs incl. zero padding of d
        kernel_name = "k_orbit<FAM_LIN, OUT_EXPABS> (liblq.so)"
        unit_txt = (f"unit = chain of {ORB_M} mirrored point pairs; per pair {TERM_FLOPS}*d + 2*{FLOPS_PER_POINT} "
                    "flop (SURVEY §8d per-coordinate term of exp-abs-linear, the coordinate division being "
                    "folded into the coefficient; one linear form serves the pair; two outer evaluations)")
    else:
        forms = my_units
        alg_flops = forms * (FLOPS_PER_PD * d + FLOPS_PER_POINT)
        conv_flops = alg_flops
        exec_flops = forms * 2 * d
        kernel_name = "k_fam<FAM_LIN, OUT_EXPABS> (liblq.so)"
        unit_txt = f"unit = point; {FLOPS_PER_PD}*d + {FLOPS_PER_POINT} flop (SURVEY §8d)"
    achieved = alg_flops / (avg_kern * 1e-3) / 1e12
    conv = conv_flops / (avg_kern * 1e-3) / 1e12
    executed = exec_flops / (avg_kern * 1e-3) / 1e12

    # e2e: the public drop-in API (host lowering, parameter upload, kernel,
    # exchange, result D2H); multi-GPU through distributed.slr_integrate
    from paper_2404_08867_b200 import distributed
    api = lq.slr_integrate if world == 1 else distributed.slr_integrate
    api(f, rule)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    xfer0 = [C.c_int64() for _ in range(3)]
    N.check(h.lq_ctx_transfer_bytes(ctx, *[C.byref(x) for x in xfer0]))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = api(f, rule)
    e2e_s = time.perf_counter() - t0
    xfer1 = [C.c_int64() for _ in range(3)]
    N.check(h.lq_ctx_transfer_bytes(ctx, *[C.byref(x) for x in xfer1]))
    h2d, d2h, params = [(b.value - a.value) / args.steps for a, b in zip(xfer0, xfer1)]
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # bytes counted by liblq at its cudaMemcpy calls (lq_ctx_transfer_bytes):
    # the coefficient upload and the 8-byte result per call; the FFT launch's
    # parameter struct (FftHead, passed by value) is reported beside them
    e2e = {"value": args.steps * n / e2e_s, "unit": "f-evals/s",
           "h2d_bytes_per_step": h2d + params, "d2h_bytes_per_step": d2h,
           "h2d_breakdown": {"cudaMemcpy": h2d, "kernel_params": params},
           "cold_first_call_ms": cold_ms, "cold_first_call_estimate": cold_est,
           "api": ("paper_2404_08867_b200.slr_integrate(f, rule)" if world == 1
                   else "paper_2404_08867_b200.distributed.slr_integrate(f, rule)"),
           "estimate": r.value}

    # MDI-LR time-to-solution on all N ranks (distributed.mdi_lr: every
    # branch's device work sharded, one exchange; max over ranks)
    mdi_dist = {}
    if world > 1 and not args.no_mdi:
        jobs = [(f"cfg{cid}", make_config(cid)) for cid in (2, 4, 5)]
        for tag, mc in jobs:
            g = lq.parse(mc.text, mc.d)
            distributed.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n)
            best = math.inf
            for _ in range(5):
                dist.barrier()
                t0 = time.perf_counter()
                v, rep = distributed.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, with_report=True)
                dt = time.perf_counter() - t0
                t = torch.tensor([dt], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                best = min(best, float(t.item()))
            mdi_dist[f"{tag}_ms"] = best * 1e3
            mdi_dist[f"{tag}_method"] = rep.method
            mdi_dist[f"{tag}_log_mean"] = rep.log_raw - rep.log_total

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    traffic = prof.get({N.LAYOUT_ORBIT_FFT: "k_orbit_fft_dram_bytes_per_launch",
                        N.LAYOUT_ORBIT: "k_orbit_dram_bytes_per_launch"}.get(lay.mode, "k_lin_dram_bytes_per_launch"))

    cpu = None
    if world == 1 and args.cpu_sample > 0:
        rate, dt, kind, what = ref_rate(args.cpu_sample, 1)
        cpu = {"value": rate, "unit": "f-evals/s", "cores": 1, "kind": kind,
               "sample": f"first {args.cpu_sample} points of cfg5 ({what}), {dt:.1f} s on 1 core; "
                         f"{os.cpu_count()} host cores, numpy {np.__version__}",
               "cpu_model": cpu_model(), "host_cores": os.cpu_count()}

    mdi = {}
    if not args.no_mdi and world == 1:
        for cid in (1, 2, 4, 5):
            mc = make_config(cid)
            g = lq.parse(mc.text, mc.d)
            mcfg = lq.MdiConfig(direct_cap=10**10) if cid == 1 else None   # as the reference needs (a^3 > 1e8)
            lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, cfg=mcfg)
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                v, rep = lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, cfg=mcfg, with_report=True)
                ts.append(time.perf_counter() - t0)
            mdi[f"cfg{cid}_ms"] = min(ts) * 1e3
            mdi[f"cfg{cid}_mean"] = rep.mean
            mdi[f"cfg{cid}_log_mean"] = rep.log_raw - rep.log_total
            mdi[f"cfg{cid}_method"] = rep.method
        # the level collapse of a non-separable integrand (suite test7's invpow,
        # d = 10, n = 8^10 + 1): the reference needs minutes (its time from the
        # build container is frozen in tests/golden/linform.json)
        g = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 10)
        lq.mdi_lr(g, 10, 8, 8**10 + 1)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            v, rep = lq.mdi_lr(g, 10, 8, 8**10 + 1, with_report=True)
            ts.append(time.perf_counter() - t0)
        mdi["invpow_d10_ms"] = min(ts) * 1e3
        mdi["invpow_d10_value"] = v
        mdi["invpow_d10_method"] = rep.method
        try:
            with open(os.path.join(REPO, "tests", "golden", "linform.json")) as fh:
                ref10 = next(c for c in json.load(fh)["cases"] if c["tag"] == "invpow_d10")
            mdi["invpow_d10_reference_s"] = ref10["ref_seconds"]
            mdi["invpow_d10_reference_value"] = float.fromhex(ref10["value"])
            mdi["invpow_d10_reference_note"] = "reference mdi_lr timed in the build container (not this box)"
        except (OSError, StopIteration, KeyError):
            pass
        # the small BASELINE plain-sum configs (parity cases; launch/latency bound)
        for cid in (1, 2, 3):
            pc = make_config(cid)
            g = lq.parse(pc.text, pc.d)
            prule = lq.korobov_vector(pc.plain_a, pc.plain_n, pc.d)
            lq.slr_integrate(g, prule)
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                lq.slr_integrate(g, prule)
                ts.append(time.perf_counter() - t0)
            mdi[f"plain_cfg{cid}_e2e_ms"] = min(ts) * 1e3
        if not args.no_ref_suite:
            # the reference as is, same box, same run (baseline/_ref; one core each)
            ref = reference_suite()
            if ref is None:
                mdi["reference"] = "baseline/_ref not installed on this box"
            else:
                mdi["reference"] = ref
                for key, ours in (("slr_cfg1_s", "plain_cfg1_e2e_ms"), ("slr_cfg2_s", "plain_cfg2_e2e_ms"),
                                  ("slr_cfg3_s", "plain_cfg3_e2e_ms"), ("mdi_cfg2_s", "cfg2_ms"),
                                  ("mdi_cfg1_s", "cfg1_ms")):
                    if key in ref:
                        mdi[f"speedup_{key[:-2]}"] = ref[key] / (mdi[ours] * 1e-3)
                mdi["reference_cores"] = "1 core per config (5 processes side by side)"

    line = {
        "metric": METRIC, "value": value, "unit": "f-evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config 5)",
        "config": {"workload": "cfg5_plain_sum", "d": d, "n": n, "a": cfg.plain_a,
                   "integrand": "exp(-|sum c_j (x_j - w_j)|)", "parallelism": f"index-range x{world}",
                   "l2": "flushed between timed steps (256 MiB write); working set 16 KB (compute-bound)"},
        "estimate": estimate,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "kernel": kernel_name, "kernel_ms": avg_kern,
                     "layout": {N.LAYOUT_ORBIT_FFT: "orbit-fft", N.LAYOUT_ORBIT: "orbit",
                                N.LAYOUT_PAIRED: "paired"}.get(lay.mode, "index"),
                     "flops_per_unit": unit_txt,
                     "survey_convention": {"achieved": conv, "frac": conv / fp64_peak,
                                           "note": ("3 flop per point-dim (incl. the coordinate division r/n) "
                                                    "charged once per linear form"
                                                    + ("; i.e. what the direct O(d) evaluation of the same linear "
                                                       "forms would have to sustain" if lay.mode == N.LAYOUT_ORBIT_FFT
                                                       else ""))},
                     "fp64_pipe_busy_ncu": prof.get({N.LAYOUT_ORBIT_FFT: "k_orbit_fft", N.LAYOUT_ORBIT: "k_orbit"}
                                                    .get(lay.mode, "k_fam_index_kernel"), {}).get("fp64_pipe_pct_of_peak"),
                     # integer work is not counted in flops; its pipe shares beside FP64's
                     "pipes_pct_ncu": prof.get({N.LAYOUT_ORBIT_FFT: "k_orbit_fft", N.LAYOUT_ORBIT: "k_orbit"}
                                               .get(lay.mode, "k_fam_index_kernel"), {}).get("pipes_pct_of_peak"),
                     "executed_dfma_tflops": executed, "executed_frac": executed / fp64_peak,
                     "peak_source": "measured in-run by lq_fp64_peak (DFMA chains, ~1 s); "
                                    "MEASURED_PEAKS.json has no FP64 entry"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "mdi_lr_time_to_solution": mdi if world == 1 else {"ranks": world, **mdi_dist},
        "notes": ("workload = BASELINE config 5 plain sum (largest single-GPU config; configs 1-3 are "
                  "sub-millisecond parity cases, timed end to end under mdi_lr_time_to_solution.plain_*); "
                  "roofline bound is the FP64 pipe (no tensor-core or HBM-bound work on this path)"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
