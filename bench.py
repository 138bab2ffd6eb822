#!/usr/bin/env python
"""SAA samples/sec for risk(z) + grad_risk(z) through the MR-DINO surrogate
on B200 (BASELINE.json metric), default workload = BASELINE config 2:
elliptic 2D 129x129, MLP 228->512x4->128 (ELU, residual), N=16384 samples
per GPU, one step = mean+variance AND exact CVaR_0.95 risk + gradient.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--config c1..c4] [--scaling weak|strong]

One process per GPU (torchrun for N>1, NCCL).  c1/c2: per-GPU work fixed
(weak scaling, the config's N per GPU); c3/c4: the config's global N is
sharded over the GPUs (strong scaling, as BASELINE specifies them).
`value` = all ranks' samples / max-over-ranks device time, the same outer
CUDA-event timer at every GPU count.  See DESIGN.md section "Measurement"
for every field.
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

METRIC = "SAA samples/sec for risk+grad_risk(z)"
JAC_METRIC = "batched control-Jacobian samples/sec (dq/dz decoded to d_u x d_z)"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--gemm", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-samples", type=int, default=8192, help="bounded CPU-baseline sample (~10-20 s)")
    ap.add_argument("--ref-samples", type=int, default=1024,
                    help="--impl reference: samples per timed step (a bounded sample of the workload)")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="weak: the config's N per GPU; strong: the config's N over all GPUs "
                         "(auto: strong for c3/c4, which BASELINE specifies sharded over 8 GPUs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


DTYPE = "f32 (bf16x3 tensor-core products, fp32 accumulate; fp64 QoI, moments and reductions)"


def scaling_mode(args):
    if args.scaling != "auto":
        return args.scaling
    return "strong" if args.config in ("c3", "c4") else "weak"


def shard_of(cfg, mode, world, rank):
    """(n_global, start, count) of this rank's contiguous sample shard."""
    from paper_2305_20053_b200.distributed import shard_range
    if mode == "weak":
        n_global = cfg.n_samples * world
        return n_global, rank * cfg.n_samples, cfg.n_samples
    a, b = shard_range(cfg.n_samples, world, rank)
    return cfg.n_samples, a, b - a


def config_block(cfg, mode, world, risks):
    """The workload description; identical for both arms (--impl ours / reference)."""
    n_global = cfg.n_samples * world if mode == "weak" else cfg.n_samples
    return {"workload": cfg.name, "description": cfg.description, "global_samples": n_global,
            "samples_per_gpu": n_global // world if n_global % world == 0 else n_global / world,
            "risks": [f"{r['kind']}(beta={r['beta']})" for r in risks], "alpha": cfg.alpha,
            "parallelism": f"dp{world} sample shards", "scaling": mode}


def risks_for(cfg):
    out = []
    for r in cfg.risks:
        d = dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha)
        out.append(d)
    return out


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.stamps = []
        self.t0 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i",
                 str(self.device), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.stamps.append(time.monotonic())
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 3.0):
        """Block until nvidia-smi has delivered its first sample (its start-up --
        NVML initialisation, device enumeration -- takes driver locks for tens of
        milliseconds; a timed region that begins meanwhile sees launch stalls)."""
        t_end = time.monotonic() + timeout
        while self.proc and not self.lines and time.monotonic() < t_end:
            time.sleep(0.01)

    def mark(self):
        """Start of the timed region: summary() uses the samples taken from here on."""
        self.t0 = time.monotonic()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.lines:
            return None
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.t0 is not None:
            timed = [ln for ts, ln in zip(self.stamps, self.lines) if ts >= self.t0]
            lines = timed or self.lines
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1", "0x1"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle port, forward-mode Jacobian as
# ouukit's SurrogateEvaluator) on a bounded sample of the same workload


def cpu_reference_rate(cfg, seed, n_cpu, reps=1, chunk=512):
    """The reference evaluator's chunked loop (riskopt.py:178-194, chunk = 512
    samples) over n_cpu samples, then the risks on the concatenated (Q, G)."""
    from oracle import mrdino_ref as ref
    from paper_2305_20053_b200 import workloads as wl
    p = wl.make_problem(cfg.with_samples(n_cpu), seed=seed, count=n_cpu)
    m = ref.as_oracle(p)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    z = p.z.astype(np.float64)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        parts = [ref.evaluate_forward_mode(m, p.m_r[a:a + chunk], z, form) for a in range(0, n_cpu, chunk)]
        Q = np.concatenate([q for q, _ in parts])
        G = np.concatenate([g for _, g in parts])
        for r in cfg.risks:
            ref.saa_objective(Q, G, z, ref.Risk(r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha),
                              t=float(np.quantile(Q, r.beta)) if r.kind == "cvar" else None)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return n_cpu / best, best


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    """CPU model name of the host the CPU legs ran on (BASELINE.md section 4 asks for it)."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference's own CPU algorithm -- the forward-mode
    chunked SurrogateEvaluator loop + saa_objective (riskopt.py:163-243),
    restated in oracle/ (fp64 numpy, all BLAS threads) because the reference
    package cannot travel to the GPU box -- on this workload.  Each step is a
    bounded sample (--ref-samples) of the workload's samples; its cost is
    linear in N, so samples/s is the workload's rate.  Rank 0 only."""
    if rank != 0:
        return
    mode = scaling_mode(args)
    n_step = min(args.ref_samples, cfg.n_samples)
    from oracle import mrdino_ref as ref
    from paper_2305_20053_b200 import workloads as wl
    p = wl.make_problem(cfg.with_samples(n_step), seed=args.seed, count=n_step, with_decoder=cfg.jacobian)
    m = ref.as_oracle(p)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    z = p.z.astype(np.float64)
    chunk = 512

    def step():
        if cfg.jacobian:                   # c5: z_jacobian_batch + decode (test_acceptance.py:326)
            Z = np.broadcast_to(z, (n_step, cfg.d_z))
            for a in range(0, n_step, 256):
                np.einsum("du,iuk->idk", p.U.astype(np.float64), ref.z_jacobian_batch(m, p.m_r[a:a + 256], Z[a:a + 256]))
            return
        parts = [ref.evaluate_forward_mode(m, p.m_r[a:a + chunk], z, form) for a in range(0, n_step, chunk)]
        Q = np.concatenate([q for q, _ in parts])
        G = np.concatenate([g for _, g in parts])
        for r in cfg.risks:
            ref.saa_objective(Q, G, z, ref.Risk(r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha),
                              t=float(np.quantile(Q, r.beta)) if r.kind == "cvar" else None)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = n_step * args.steps / dt
    sample = (f"{n_step} of the workload's {cfg.n_samples} samples per step, in the reference evaluator's "
              f"{chunk}-sample chunks (forward-mode z-Jacobian, fp64 numpy BLAS, {cpu_cores()} threads); "
              f"cost is linear in N")
    line = {
        "metric": JAC_METRIC if cfg.jacobian else METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": mode, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": config_block(cfg, mode, world, risks_for(cfg)),
        "samples_per_timed_step": n_step,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# BASELINE config 5: batched control Jacobian decoded to d_u x d_z


def cpu_jacobian_rate(cfg, seed, n_cpu):
    """The reference's z_jacobian_batch (surrogate.py:195-233, forward mode,
    restated in oracle/, fp64 numpy BLAS) + the decode modes @ J
    (test_acceptance.py:326) on n_cpu samples."""
    from oracle import mrdino_ref as ref
    from paper_2305_20053_b200 import workloads as wl
    p = wl.make_problem(cfg.with_samples(n_cpu), seed=seed, count=n_cpu, with_decoder=True)
    m = ref.as_oracle(p)
    Z = np.broadcast_to(p.z.astype(np.float64), (n_cpu, cfg.d_z))
    U = p.U.astype(np.float64)
    t0 = time.perf_counter()
    for a in range(0, n_cpu, 256):
        J = ref.z_jacobian_batch(m, p.m_r[a:a + 256], Z[a:a + 256])
        np.einsum("du,iuk->idk", U, J)
    dt = time.perf_counter() - t0
    return n_cpu / dt, dt


def run_jacobian(args, cfg, rank, world, local_rank, dist):
    """c5: one step = the decoded control Jacobians of this rank's samples at
    the control z, written to a device buffer (sdn_jacobian_samples).  The
    dominant cost is writing n x d_u x d_z fp32 (HBM-write bound)."""
    import torch
    from paper_2305_20053_b200 import Engine, workloads as wl
    mode = scaling_mode(args)
    n_global, start, n_loc = shard_of(cfg, mode, world, rank)
    p = wl.make_problem(cfg, seed=args.seed, start=start, count=n_loc, with_decoder=True)
    eng = Engine(p, max_samples=n_loc, device=local_rank, gemm=args.gemm)
    stream = torch.cuda.Stream(device=local_rank)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    eng.set_tracking(p.c, p.q0)
    eng.set_decoder(p.U, p.ubias, p.Mdiag_u, p.u_target)
    eng.set_samples(torch.from_numpy(p.m_r).cuda(), global_offset=start)
    z = p.z.astype(np.float64)
    J = torch.empty((n_loc, cfg.d_u, cfg.d_z), dtype=torch.float32, device="cuda")   # 1.78 GB at c5 (> L2)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        eng.jacobian_samples(z, decoded=True, out=J)
    barrier()
    launches0 = eng.kernel_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier()
        for i in range(args.steps):
            starts[i].record(stream)
            eng.jacobian_samples(z, decoded=True, out=J)   # output 1.78 GB > L2: no flush needed
            ends[i].record(stream)
        barrier()
    launches = eng.kernel_launches() - launches0
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    value = n_global * args.steps / (ms_total / 1e3)
    out_bytes = n_loc * cfg.d_u * cfg.d_z * 4

    # per-class profile (tangent GEMMs, decode GEMM)
    eng.profile(True)
    for _ in range(args.steps):
        eng.jacobian_samples(z, decoded=True, out=J)
    torch.cuda.synchronize()
    prof = eng.profile_read()
    eng.profile(False)

    # e2e: the reference-facing batch API with host buffers (m_r, z rows up;
    # the decoded Jacobians down into pinned host memory)
    Jh = torch.empty((n_loc, cfg.d_u, cfg.d_z), dtype=torch.float32).pin_memory().numpy()
    Z = np.ascontiguousarray(np.broadcast_to(p.z, (n_loc, cfg.d_z)).astype(np.float32))
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        Jh[...] = eng.jacobian_batch(p.m_r, Z, decoded=True)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n_global * e2e_steps / float(te.item())

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_bw = peaks.get("hbm_gbs", 6650.0)
    peak_src = "of measured HBM copy (MEASURED_PEAKS.json)" if peaks else "of fallback (B200_PROFILING.md)"
    step_gbps = out_bytes * args.steps / (ms / 1e3) / 1e9
    dec = prof.get("decode_gemm", {"ms": 0.0, "launches": 0})
    step_ms_prof = sum(v["ms"] for v in prof.values())
    if dec["launches"]:
        achieved = out_bytes * args.steps / (dec["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak_bw, "unit": "GB/s", "frac": achieved / peak_bw,
                "traffic": None, "kernel": "decode_gemm (tcgen05, scatter epilogue into J[i, u, k])",
                "launches": dec["launches"], "avg_launch_us": 1e3 * dec["ms"] / dec["launches"],
                "share_of_step": dec["ms"] / step_ms_prof, "algorithmic_bytes_per_launch": out_bytes,
                "peak_source": peak_src, "whole_step_GBps": step_gbps,
                "note": "achieved = decoded Jacobian bytes written (n x d_u x d_z x 4 = 108,900 B/sample) / the "
                        "decoder GEMM's launch time; whole_step_GBps divides by the whole step"}
    else:
        roof = {"bound": "hbm", "achieved": step_gbps, "peak": peak_bw, "unit": "GB/s",
                "frac": step_gbps / peak_bw, "traffic": None, "kernel": "whole Jacobian step",
                "algorithmic_bytes_per_step": out_bytes, "peak_source": peak_src}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_cpu = min(args.cpu_samples, 1024)
        rate, secs = cpu_jacobian_rate(cfg, args.seed, n_cpu)
        cpu = {"value": rate, "unit": "samples/s", "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "port",
               "sample": f"{n_cpu} samples of c5: forward-mode z_jacobian_batch in 256-sample chunks + decode "
                         f"(oracle port, fp64 numpy BLAS) ({secs:.1f} s)"}
    if rank == 0:
        line = {
            "metric": JAC_METRIC, "value": value,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "timing": "CUDA events on the launch stream around each step, max over ranks",
            "scaling": mode, "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": cfg.name, "description": cfg.description, "global_samples": n_global,
                       "samples_per_gpu": n_loc, "output_bytes_per_gpu": out_bytes,
                       "parallelism": f"dp{world} sample shards", "scaling": mode},
            "l2": "output (1.78 GB per step) larger than L2",
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": int(p.m_r.nbytes + Z.nbytes),
                    "d2h_bytes_per_step": int(out_bytes),
                    "api": "Engine.jacobian_batch (host m_r, z rows in; decoded Jacobians to pinned host memory)"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "kernel_classes": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps}
                               for k, v in prof.items() if v["launches"]},
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


ENC_METRIC = "KLE encoder fields/sec (m_r = V_m^T M (m - mean))"


def run_encoder(args, rank, world, local_rank):
    """--config enc: the cold encoder (randfield.py:67-72) on the
    c4 field shapes (d_m = 35937, r_m = 256) over a bounded number of fields --
    setup work, once per SAA sample set.  value: fields already in HBM; e2e:
    host fields in (pinned) through the public call.  Roofline: the fields are
    read once (4 d_m bytes each), so the HBM figure is the algorithmic bound;
    the kernel itself is tensor-core work: both operands split into three bf16
    planes, four bf16x3 GEMM passes per 1024-column K chunk (the fp32 product to
    ~2^-24, which the input whitening needs), fp64 accumulation across chunks."""
    import torch
    from paper_2305_20053_b200 import Engine, workloads as wl
    cfg = wl.WORKLOADS["c4"]
    n = 16384                                      # one full tensor-core pass of the encoder (2.36 GB of fields)
    p = wl.make_problem(cfg.with_samples(n), seed=args.seed)
    psi, lam, mdiag = wl.kl_modes(cfg, args.seed)
    Vm = np.ascontiguousarray(psi[:, :cfg.r_m], dtype=np.float32)
    eng = Engine(p, max_samples=n, device=local_rank, gemm=args.gemm)
    stream = torch.cuda.Stream(device=local_rank)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(args.seed)
    # synthetic fields with the KL law's scale: mean + unit-variance nodal noise (values do not change the cost)
    F = (wl.M_MEAN + torch.randn((n, cfg.d_m), generator=g, device="cuda", dtype=torch.float32)).contiguous()
    in_bytes = n * cfg.d_m * 4                     # 2.36 GB > L2
    for _ in range(max(args.warmup, 3)):
        eng.encode_fields(F, Vm, mdiag, wl.M_MEAN)
    steps = max(1, min(args.steps, 10))
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches0 = eng.kernel_launches()
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        for i in range(steps):
            starts[i].record(stream)
            eng.encode_fields(F, Vm, mdiag, wl.M_MEAN)
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = eng.kernel_launches() - launches0
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    value = n * steps / (ms / 1e3)
    Fh = F.cpu().pin_memory().numpy()
    t0 = time.perf_counter()
    for _ in range(2):
        eng.encode_fields(Fh, Vm, mdiag, wl.M_MEAN)
    e2e_value = n * 2 / (time.perf_counter() - t0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_bw = peaks.get("hbm_gbs", 6650.0)
    gbps = in_bytes * steps / (ms / 1e3) / 1e9
    flops = 2.0 * n * cfg.d_m * cfg.r_m
    line = {
        "metric": ENC_METRIC, "value": value, "unit": "fields/s", "n_gpus": world, "steps": steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / steps, "higher_is_better": True,
        "timing": "CUDA events on the launch stream around each encode call", "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 products from three-way bf16 splits (tcgen05), f64 accumulation across K chunks",
        "data": "synthetic",
        "config": {"workload": "enc", "description": f"cold KLE encoder on c4 field shapes: d_m={cfg.d_m}, "
                   f"r_m={cfg.r_m}, {n} fields per step ({in_bytes / 1e6:.0f} MB > L2; c4's full set is 18.8 GB)",
                   "fields_per_step": n, "parallelism": "dp1"},
        "l2": "inputs larger than L2 (2.36 GB per step)",
        "e2e": {"value": e2e_value, "unit": "fields/s", "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": 0, "api": "Engine.encode_fields (host fields in; m_r stays on the device)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": gbps, "peak": peak_bw, "unit": "GB/s", "frac": gbps / peak_bw,
                     "traffic": None, "kernel": "tc_gemm_kernel<EpiAccum64> x 4 passes per K chunk (+ k_split3)",
                     "algorithmic_bytes_per_step": in_bytes,
                     "fp32_tflops": flops * steps / (ms / 1e3) / 1e12,
                     "note": "algorithmic bytes = the fields read once; the work is 2 n d_m r_m flops x 12 bf16 MMAs "
                             "per product (tensor bound), plus the split's 6 B written per field value"},
        "cpu_baseline": None, "clocks": clk.summary(),
    }
    print(json.dumps(line))


def main():
    args = parse()
    if args.config == "enc":
        if args.impl == "reference" or int(os.environ.get("WORLD_SIZE", "1")) > 1:
            print(json.dumps({"impl": args.impl, "unavailable": "enc is a single-GPU setup benchmark of this repo only"}))
            return
        import torch
        torch.cuda.set_device(0)
        run_encoder(args, 0, 1, 0)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2305_20053_b200 import workloads as wl
    cfg = wl.WORKLOADS[args.config]

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    if cfg.jacobian:
        run_jacobian(args, cfg, rank, world, local_rank, dist)
        return

    from paper_2305_20053_b200 import Engine
    mode = scaling_mode(args)
    n_global, start, n_loc = shard_of(cfg, mode, world, rank)
    p = wl.make_problem(cfg, seed=args.seed, start=start, count=n_loc)
    eng = Engine(p, max_samples=n_loc, device=local_rank, gemm=args.gemm)
    # one non-default stream for the engine, the L2 flush, the timing events
    # and (N > 1) NCCL: events on it order with the engine's graph launches
    stream = torch.cuda.Stream(device=local_rank)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(torch.from_numpy(p.m_r).cuda(), global_offset=start)   # resident in HBM
    risks = risks_for(cfg)
    z = p.z.astype(np.float64)
    for d in risks:
        if d["kind"] == "cvar":
            # smoothed CVaR: t starts at the beta-VaR of Q(z0), as the reference's
            # minimize initialises it (riskopt.py:295-297); rank 0's value for all
            from paper_2305_20053_b200.api import mc_var
            q0, _ = eng.eval_samples(z, need_grad=False)
            tt = torch.tensor([mc_var(q0, d["beta"])], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.broadcast(tt, 0)
            d["t"] = float(tt.item())
    sharded = None
    if world > 1:
        from paper_2305_20053_b200.distributed import ShardedObjective, TorchComm
        sharded = ShardedObjective(eng, TorchComm(dist), n_global=n_global)

    def step(end_event=None):
        """One evaluation; end_event (if given) is recorded on the stream right
        after the device work is enqueued, before the host reads the results."""
        if sharded is not None:
            res = sharded.eval_multi(z, risks)
            if end_event is not None:
                end_event.record(stream)
            return res
        eng.eval_multi_launch(z, risks)
        if end_event is not None:
            end_event.record(stream)
        return eng.eval_multi_wait()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    # the clock sampler starts ahead of the warm-up: nvidia-smi's start-up (NVML initialisation) holds driver locks
    # for tens of ms, which a timed region beginning right behind it would see as launch stalls; its samples count
    # from clk.mark() on
    with ClockSampler(local_rank) as clk:
        for _ in range(max(args.warmup, 3)):
            step()
        barrier()
        clk.wait_first()

        # ---- timed region: device time per step (CUDA events on the engine's stream)
        launches0 = eng.kernel_launches()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        barrier()
        clk.mark()
        dev_steps = []
        for i in range(args.steps):
            flush.zero_()                     # L2 flush between steps (untimed)
            starts[i].record(stream)
            res = step(ends[i])
            if sharded is None:
                dev_steps.append(eng.last_device_ms())
        barrier()
    launches = eng.kernel_launches() - launches0
    per_step_outer = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # the same timer at every GPU count: CUDA events on the launch stream
    # around each step (device work, NCCL exchanges and any host staging gaps
    # between them; the end event is enqueued behind the step's last device
    # work, so the host's wake-up to read the results is not in it).  N = 1
    # also reports the engine's in-graph device span (graph's first to last
    # node) beside it.
    per_step = per_step_outer
    ms = sum(per_step)
    if os.environ.get("SDN_BENCH_STEPS_DUMP"):
        print("per-step ms:", " ".join(f"{x:.4f}" for x in per_step), file=sys.stderr)
    t_local = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_total = float(t_local.item())
    ms_step = ms_total / args.steps
    value = n_global * args.steps / (ms_total / 1e3)

    # ---- profiled pass (same steps, per-launch events by kernel class)
    eng.profile(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = eng.profile_read()
    eng.profile(False)

    # ---- e2e through the public API with host buffers (wall clock incl. H2D/D2H)
    from paper_2305_20053_b200 import _lib
    barrier()
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()                      # L2 flushed between steps, outside the timed call
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = step()                       # host z in -> device -> host value/grad/indices out
        e2e_s += time.perf_counter() - t0
    t_e2e = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = n_global * args.steps / float(t_e2e.item())
    kmax = sum(max(int(np.ceil((1 - r["beta"]) * n_global - 1e-9)), 1) for r in risks
               if r["kind"] == "cvar_exact")
    h2d = 8 * cfg.d_z
    # results read back per step: moments + each risk's partials (fp64), and
    # the exact-CVaR selection (int32 local indices on one GPU; the merged
    # global candidate set, fp64 global index + mask byte, when sharded)
    idx_bytes = 4 * kmax if world == 1 else 9 * world * kmax
    d2h = len(risks) * 8 * (_lib.STATS_LEN + eng.partial_len()) + idx_bytes

    # ---- roofline of the dominant kernel class
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    # the timed loop is short (K steps of well under a second): the burst peak applies
    peak_tf = peaks.get("bf16_tflops", 1590.0)
    peak_src = "of measured bf16 burst (MEASURED_PEAKS.json)" if peaks else "of fallback (B200_PROFILING.md)"
    dom = max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    step_ms_prof = sum(v["ms"] for v in prof.values())
    if d["flops"] > 0:
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf, "traffic": None, "kernel": dom,
                "launches": d["launches"], "avg_launch_us": 1e3 * d["ms"] / max(d["launches"], 1),
                "share_of_step": d["ms"] / step_ms_prof, "peak_source": peak_src,
                "frac_of_bf16x3_effective": achieved / (peak_tf / 3.0),
                "frac_of_sustained": achieved / peaks.get("bf16_tflops_sustained", peak_tf),
                "note": "achieved = algorithmic flops (2 per MAC, no bf16x3 factor) / class time; every "
                        "product issues 3 bf16 MMAs, so the attainable ceiling is peak/3"}
    else:
        bw = d["bytes"] / (d["ms"] / 1e3) / 1e9
        peak_bw = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": bw, "peak": peak_bw, "unit": "GB/s", "frac": bw / peak_bw,
                "traffic": None, "kernel": dom, "launches": d["launches"],
                "share_of_step": d["ms"] / step_ms_prof, "peak_source": peak_src}
    tf_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf_path):
        try:
            roof["traffic"] = json.load(open(tf_path)).get(args.config, {}).get(dom)
        except Exception:
            pass

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, secs = cpu_reference_rate(cfg, args.seed, args.cpu_samples, reps=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "port",
               "sample": f"{args.cpu_samples} samples of {cfg.name} in the reference evaluator's 512-sample "
                         f"chunks, forward-mode z-Jacobian (oracle port, fp64 numpy BLAS), all of the "
                         f"workload's risks ({secs:.1f} s)"}

    if rank == 0:
        per_class = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps}
                     for k, v in prof.items() if v["launches"]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "timing": "CUDA events on the launch stream: start before each step's host staging, end enqueued behind its last device work (every N; N>1 includes the exchanges and host phase gaps), max over ranks",
            "ms_per_step_device_span": (sum(dev_steps) / args.steps) if dev_steps else None,
            "ms_per_step_median": float(np.median(per_step)),
            "scaling": mode, "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": config_block(cfg, mode, world, risks),
            "gemm": args.gemm, "l2": "flushed between steps (256 MiB write, untimed)",
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "Engine.eval_multi (host z in, host value/grad/indices out)"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "kernel_classes": per_class,
            "clocks": clk.summary(),
        }
        one_launch = (world == 1 and launches <= 3 * args.steps and args.gemm == "auto")
        if one_launch:
            # small sample sets run the whole evaluation in one launch (csrc/small.cuh, fp32 FFMA);
            # the per-class profile above is the layer-by-layer path (profiling disables the one-launch path)
            line["dtype"] = "f32 (FFMA; fp64 QoI, moments and reductions)"
            line["path"] = "one evaluation kernel (k_small_eval) + the z fetch per evaluation; kernel_classes/roofline: the layer-by-layer path"
            flops = cfg.flops_forward() + cfg.flops_backward() if hasattr(cfg, "flops_backward") else None
            if flops and dev_steps:
                line["one_launch_tflops"] = flops * n_loc / (sum(dev_steps) / args.steps / 1e3) / 1e12
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
