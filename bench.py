#!/usr/bin/env python
"""Benchmark of the B200 projected star-Q / tSVDQ engine (BASELINE.json metric:
"tSVDQ input GB/s and star-Q product TFLOP/s (FP64) vs roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5|cfg4|cfg3|cfg2]
                  [--impl ours|reference]

Workloads (BASELINE.json configs, synthetic inputs of the named shapes):
  cfg5  2048x2048x1024 rank-50 CP + noise; data-driven Q (p=128) + tSVDQ k=32
        + fused reconstruction relative error.  metric: tSVDQ input GB/s.
  cfg4  star-Q product A 1024x512x256 * B 512x1024x256, DCT p=64.  metric: TFLOP/s.
  cfg3  512x512x224 hyperspectral, data Q p=32, k=16.  cfg2  240x320x200 video, p=20, k=10.

One step = one pass of the hot path over one input already resident in HBM
(`value`); `e2e` repeats it through the C-ABI with pinned HOST buffers, the
H2D of the inputs and the D2H of the result inside the timed region.
Under torchrun (N>1) cfg5 is pixel-sharded across the ranks (dist.py; strong
scaling, one global tensor); the other workloads run one independent instance
per rank (weak scaling, no data-path collective).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_FALLBACK = 36.914  # TFLOP/s, MEASURED_FP64.json (DMMA m8n8k4, this pool)


def load_peaks():
    """Roofline denominators. HBM and bf16 come from the driver-written
    MEASURED_PEAKS.json; FP64 (DMMA) from MEASURED_FP64.json (tools/fp64_peaks.cu
    on this pool: there is no FP64 tcgen05 kind, so the driver's bf16 GEMM says
    nothing about it); dense INT8 is taken as 2x the driver's measured bf16
    burst (the B200's dense INT8 rate is twice its bf16 rate: 4.5 vs 2.25
    POPS nominal), with cuBLASLt's measured INT8 GEMM noted beside it."""
    peaks = {"hbm_gbs": 6540.5, "fp64_tflops": FP64_PEAK_FALLBACK,
             "hbm_src": "MEASURED_PEAKS.json", "fp64_src": "MEASURED_FP64.json",
             "int8_tops": 4500.0, "int8_src": "nominal B200 dense INT8 (fallback)", "int8_cublaslt_tops": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        # the dominant kernels run inside a long step (20 back-to-back steps
        # of 130 ms), so the sustained tensor figure is the denominator
        # (B200_PROFILING.md); the burst one is reported beside it
        if mp.get("bf16_tflops_sustained"):
            peaks["int8_tops"] = 2.0 * float(mp["bf16_tflops_sustained"])
            peaks["int8_src"] = ("2 x bf16_tflops_sustained of the driver-written MEASURED_PEAKS.json "
                                 "(dense INT8 = 2x dense bf16 on B200; sustained: the kernel runs inside a "
                                 "long step)")
        if mp.get("bf16_tflops"):
            peaks["int8_burst_tops"] = 2.0 * float(mp["bf16_tflops"])
            if not mp.get("bf16_tflops_sustained"):
                peaks["int8_tops"] = peaks["int8_burst_tops"]
                peaks["int8_src"] = "2 x bf16_tflops (burst) of the driver-written MEASURED_PEAKS.json"
    except Exception:
        peaks["hbm_gbs"], peaks["hbm_src"] = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_INT8.json")) as f:
            peaks["int8_cublaslt_tops"] = float(json.load(f)["int8_tops"])
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "MEASURED_FP64.json")) as f:
            d = json.load(f)
        peaks["fp64_tflops"] = float(d.get("dmma_sustained_tflops", d["dmma_m8n8k4_tflops"]))
        peaks["fp64_src"] = "MEASURED_FP64.json dmma_sustained_tflops (tools/fp64_peaks.cu, this pool)"
    except Exception:
        peaks["fp64_src"] = "constant from MEASURED_FP64.json (r01)"
    return peaks


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self):
        """Start of the timed region: only samples written after this count.
        (nvidia-smi is started before the warm-up steps: its start-up, which
        holds the driver for a while, must not land inside the timed steps.)"""
        self.skip = 0
        if self.path:
            try:
                with open(self.path) as f:
                    self.skip = sum(1 for _ in f)
            except OSError:
                pass

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for i, line in enumerate(open(self.path)):
            if i < getattr(self, "skip", 0):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- helpers
def sync_all(dist_on):
    import torch
    torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()


def max_over_ranks(x, dist_on):
    if not dist_on:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(workload, stage):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/<round>/ncu_<stage>_<workload>_raw.csv)."""
    import csv
    import glob
    names = {"gram_syrk": "ws_syrk", "facewise": "cfg4_gemms", "ozaki_syrk": "ozaki_syrk", "ozaki_gemm": "ozaki_face"}
    key = names.get(stage, stage)
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_{key}*raw.csv")), reverse=True):
        if workload not in os.path.basename(path) and stage != "facewise":
            continue
        try:
            rows = list(csv.reader(open(path)))
            hdr, units = rows[0], rows[1]
            ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            r = rows[2]
            tot = float(r[ir].replace(",", "")) * scale.get(units[ir], 1) + \
                float(r[iw].replace(",", "")) * scale.get(units[iw], 1)
            return tot, os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def timing_report(L, reset=True):
    buf = C.create_string_buffer(1 << 16)
    rc = L.ppc_timing_report(buf, len(buf), 1 if reset else 0)
    if rc:
        raise RuntimeError(L.ppc_last_error().decode())
    return json.loads(buf.value.decode())


def ptr(t):
    return C.c_void_p(t.data_ptr())


def flat_host(t):
    """Pinned host copy of a Fortran-laid-out device tensor (mode-1 fastest)."""
    return t.permute(*reversed(range(t.dim()))).contiguous().reshape(-1).cpu().pin_memory()


# --------------------------------------------------------------- workloads
class StarQ:
    """cfg4: C = [(A x3 Q^T) facewise (B x3 Q^T)] x3 Q (star_products.cpp:51-59)."""

    name = "cfg4"
    metric, unit = "starq_tflops", "TFLOP/s"

    def __init__(self, n1=1024, m=512, n2=1024, n3=256, p=64, seed=0):
        import torch
        import paper_2409_19402_b200 as pp
        from paper_2409_19402_b200 import synth
        self.dims = (n1, m, n2, n3, p)
        self.A = synth.gaussian_device(n1, m, n3, seed, 1)
        self.B = synth.gaussian_device(m, n2, n3, seed, 2)
        self.Q = pp.to_device(pp.Transform("dct", n3, p).q)
        self.Cout = pp.empty_device((n1, n2, n3))
        self.flops = 2.0 * p * (n1 * m * n3 + m * n2 * n3 + n1 * m * n2 + n1 * n2 * n3)
        self.in_bytes = 8.0 * (n1 * m * n3 + m * n2 * n3)
        self.torch = torch

    def config(self):
        n1, m, n2, n3, p = self.dims
        return {"workload": "cfg4 star-Q product", "A": [n1, m, n3], "B": [m, n2, n3], "p": p,
                "transform": "dct", "l2": "inputs (2 GiB) > L2; no flush needed"}

    def step(self, L):
        n1, m, n2, n3, p = self.dims
        rc = L.ppc_star_q_product(ptr(self.A), n1, m, n3, ptr(self.B), n2, ptr(self.Q), p,
                                  C.c_double(1.0), ptr(self.Cout), 1)
        if rc:
            raise RuntimeError(L.ppc_last_error().decode())

    def value(self, sec):
        return self.flops / sec / 1e12

    def dominant(self, stages):
        # the single longest kernel launch of the step: the inverse transform
        # (INT8 row-split kernel, bound by its 8-byte FP64 stores: HBM; FP64
        # DMMA where not eligible), the facewise product (INT8 Ozaki MMA when
        # eligible) or a forward transform (FP64 DMMA)
        cands = [("ozaki_star_inv", "hbm") if "ozaki_star_inv" in stages else ("mode3_inv", "tensor"),
                 ("ozaki_gemm", "int8") if "ozaki_gemm" in stages else ("facewise", "tensor"),
                 ("mode3_fwd", "tensor")]
        cands = [c for c in cands if c[0] in stages]
        if not cands:
            return ("facewise", "tensor")
        return max(cands, key=lambda c: stages[c[0]]["ms"] / max(1, stages[c[0]]["n"]))

    def e2e_setup(self):
        torch = self.torch
        n1, m, n2, n3, p = self.dims
        self.hA = flat_host(self.A)
        self.hB = flat_host(self.B)
        self.hQ = flat_host(self.Q)
        self.hC = torch.empty(n1 * n2 * n3, dtype=torch.float64).pin_memory()
        self.h2d = 8 * (n1 * m * n3 + m * n2 * n3 + n3 * p)
        self.d2h = 8 * n1 * n2 * n3

    def e2e_step(self, L):
        n1, m, n2, n3, p = self.dims
        rc = L.ppc_star_q_product(ptr(self.hA), n1, m, n3, ptr(self.hB), n2, ptr(self.hQ), p,
                                  C.c_double(1.0), ptr(self.hC), 0)
        if rc:
            raise RuntimeError(L.ppc_last_error().decode())

    def cpu_sample(self, ppo, threads):
        """The full cfg4 product (no cut, no extrapolation) on the oracle
        (star_products.cpp:51-59 restated), GEMMs on OpenBLAS with `threads`."""
        from paper_2409_19402_b200 import synth
        n1, m, n2, n3, p = self.dims
        a = synth.gaussian(n1, m, n3, seed=0, stream=1)
        b = synth.gaussian(m, n2, n3, seed=0, stream=2)
        q = ppo.dct_q(n3, p)
        flops = 2.0 * p * (n1 * m * n3 + m * n2 * n3 + n1 * m * n2 + n1 * n2 * n3)
        t0 = time.perf_counter()
        ppo.star_q_product(a, b, q)
        sec = time.perf_counter() - t0
        return flops / sec / 1e12, {
            "sample": f"the full cfg4 product A {n1}x{m}x{n3} * B {m}x{n2}x{n3}, p={p} (no cut), 1 rep",
            "how": f"oracle/ppo.c star_q_product, GEMMs on OpenBLAS {threads} thread(s)", "extrapolated": False,
            "seconds": sec}


_CPU_SAMPLES = {}


class Tsvdq:
    """cfg2/3/5: data-driven Q (transforms.cpp:97-115) + tsvdq (decompositions.cpp:62-83)
    + relative_error(A, tsvdq_reconstruct(F)) fused (tools/main.cpp:276-283 chain)."""

    metric, unit = "tsvdq_input_GBps", "GB/s"

    def __init__(self, name, n1, n2, n3, p, k, seed=0):
        import torch
        import paper_2409_19402_b200 as pp
        from paper_2409_19402_b200 import synth
        self.name = name
        self.dims = (n1, n2, n3, p, k)
        self.torch = torch
        if name == "cfg5":
            self.A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=seed)
        elif name == "cfg3":
            self.A = pp.to_device(synth.hyperspectral(n1, n2, n3, seed=seed))
        else:
            self.A = pp.to_device(synth.video(n1, n2, n3, seed=seed))
        self.Q = pp.empty_device((n3, p))
        self.U = pp.empty_device((n1, k, p))
        self.S = pp.empty_device((k, p))
        self.V = pp.empty_device((n2, k, p))
        self.in_bytes = 8.0 * n1 * n2 * n3
        self.re = None

    def config(self):
        n1, n2, n3, p, k = self.dims
        desc = {"cfg5": "cfg5 rank-50 CP + N(0,1e-3^2) noise", "cfg3": "cfg3 hyperspectral",
                "cfg2": "cfg2 video"}[self.name]
        if self.name == "cfg2":
            return {"workload": desc + " tSVDQ sweep with data-driven Q", "shape": [n1, n2, n3], "p": p,
                    "k": [1, 5, 10, 20],
                    "step": "ppc_tsvdq_sweep = data_dependent_transform + tsvdq + relative_error(A, recon) "
                            "for every k (tools/main.cpp:299-341 cmd_sweep), slice SVDs shared at kmax",
                    "l2": "input > L2" if self.in_bytes > 126e6 else "input < L2 (resident)"}
        return {"workload": desc + " tSVDQ with data-driven Q", "shape": [n1, n2, n3], "p": p,
                "k": k, "step": "ppc_tsvdq_compress = data_dependent_transform + tsvdq + relative_error(A, recon) (tools/main.cpp:186-283)",
                "l2": "input > L2" if self.in_bytes > 126e6 else "input < L2 (resident)"}

    def step(self, L):
        n1, n2, n3, p, k = self.dims
        if self.name == "cfg2":
            # BASELINE configs[1]: tSVDQ at k in {1, 5, 10, 20} -> the sweep
            ks = (C.c_int64 * 4)(1, 5, 10, 20)
            ps = (C.c_int64 * 1)(p)
            re = (C.c_double * 4)()
            rc = L.ppc_tsvdq_sweep(ptr(self.A), n1, n2, n3, ps, 1, ks, 4, None, re, 1)
            if rc:
                raise RuntimeError(L.ppc_last_error().decode())
            self.re = list(re)
            return
        re = C.c_double()
        rc = L.ppc_tsvdq_compress(ptr(self.A), n1, n2, n3, p, k, ptr(self.Q), None, ptr(self.U),
                                  ptr(self.S), ptr(self.V), C.byref(re), 1)
        if rc:
            raise RuntimeError(L.ppc_last_error().decode())
        self.re = re.value

    def value(self, sec):
        return self.in_bytes / sec / 1e9

    def step_given_q(self, L):
        """tsvdq(A, Q, k) alone (decompositions.cpp:62-83) with the basis the
        last compress step left in self.Q: SURVEY 8(d) asks for the tSVDQ
        time both with a given Q and including its construction."""
        n1, n2, n3, p, k = self.dims
        rc = L.ppc_tsvdq(ptr(self.A), n1, n2, n3, ptr(self.Q), p, k, ptr(self.U), ptr(self.S), ptr(self.V), 1)
        if rc:
            raise RuntimeError(L.ppc_last_error().decode())

    def dominant(self, stages):
        # the single most expensive kernel launch of the step (ncu launch
        # list: the Gram SYRK, on the INT8 tensor cores when the Ozaki path
        # runs); slice_svd is a composite of many kernels
        return ("ozaki_syrk", "int8") if "ozaki_syrk" in stages else ("gram_syrk", "tensor")

    def e2e_setup(self):
        torch = self.torch
        n1, n2, n3, p, k = self.dims
        self.hA = flat_host(self.A)
        self.hQ = torch.empty(n3 * p, dtype=torch.float64).pin_memory()
        self.hU = torch.empty(n1 * k * p, dtype=torch.float64).pin_memory()
        self.hS = torch.empty(k * p, dtype=torch.float64).pin_memory()
        self.hV = torch.empty(n2 * k * p, dtype=torch.float64).pin_memory()
        # one public call per step (ppc_tsvdq_compress, the CLI compress chain):
        # H2D of A, D2H of Q + factors + the relative error
        self.h2d = 8 * n1 * n2 * n3
        self.d2h = 8 * (n3 * p + (n1 + n2 + 1) * k * p) + 8
        if self.name == "cfg2":  # the sweep returns the RE grid only
            self.d2h = 8 * 4

    def e2e_step(self, L):
        n1, n2, n3, p, k = self.dims
        if self.name == "cfg2":
            ks = (C.c_int64 * 4)(1, 5, 10, 20)
            ps = (C.c_int64 * 1)(p)
            re = (C.c_double * 4)()
            rc = L.ppc_tsvdq_sweep(ptr(self.hA), n1, n2, n3, ps, 1, ks, 4, None, re, 0)
            if rc:
                raise RuntimeError(L.ppc_last_error().decode())
            return
        re = C.c_double()
        rc = L.ppc_tsvdq_compress(ptr(self.hA), n1, n2, n3, p, k, ptr(self.hQ), None, ptr(self.hU),
                                  ptr(self.hS), ptr(self.hV), C.byref(re), 0)
        if rc:
            raise RuntimeError(L.ppc_last_error().decode())

    def cpu_sample(self, ppo, threads):
        """cfg5: the full config (n3=1024, p=128, k=32, 2048^2 slices) on the
        LAPACK restatement (oracle/baseline.py), timed on an N/64 lateral pixel
        sample (QR, transforms, reconstruction + residual) and one whole
        2048^2 slice SVD, extrapolated linearly in N and p (BASELINE.md
        section 4). cfg2: the full video on the C oracle. cfg3: the oracle on
        a 128x128 cut of the cube (n3, p, k kept)."""
        import numpy as np
        from paper_2409_19402_b200 import synth
        n1, n2, n3, p, k = self.dims
        if self.name == "cfg5":
            from oracle import baseline
            nj = n2 // 64
            if "cfg5" not in _CPU_SAMPLES:  # generated once per process (not timed)
                _CPU_SAMPLES["cfg5"] = (synth.cp_block(n1, n2, n3, 0, nj, rank=50, noise=1e-3, seed=1),
                                        synth.cp_slice(n1, n2, rank=50, noise=1e-3, seed=1, i=0))
            blk, sl = _CPU_SAMPLES["cfg5"]
            sec, det = baseline.compress_timed(lambda w: blk, n1, n2, n3, p, k, nj, lambda i: sl)
            return (8.0 * n1 * n2 * n3) / sec / 1e9, {
                "sample": (f"full config {n1}x{n2}x{n3}, p={p}, k={k}: QR/transforms/reconstruction on a "
                           f"{n1}x{nj}x{n3} lateral pixel sample (N/64), 1 whole {n1}x{n2} slice SVD; "
                           "extrapolated linearly in N and p"),
                "how": ("reference chain restated on LAPACK/BLAS (oracle/baseline.py: dgeqrf + dgesdd for Q, "
                        "dgemm transforms, dgesdd per slice; numpy OpenBLAS, all host threads); dgesdd is far "
                        "faster than the reference's Jacobi SVD, so this CPU figure is optimistic"),
                "extrapolated": True, "seconds": sec, "parts": det}
        if self.name == "cfg3":
            s1, s2 = 128, 128
            a = synth.hyperspectral(s1, s2, n3, seed=1)
        else:
            s1, s2 = n1, n2
            a = synth.video(n1, n2, n3, seed=1)
        t0 = time.perf_counter()
        q, _, _ = ppo.data_dependent_q(a, p)
        if self.name == "cfg2":  # cmd_sweep: one tsvdq + reconstruction per k
            for kk in (1, 5, 10, 20):
                U, S, V = ppo.tsvdq(a, q, kk)
                ppo.relative_error(a, ppo.tsvdq_reconstruct(U, S, V, q))
            sec = time.perf_counter() - t0
            return (8.0 * s1 * s2 * n3) / sec / 1e9, {
                "sample": f"oracle data Q + tsvdq + RE for k in 1,5,10,20 on the full {s1}x{s2}x{n3} video (p={p})",
                "how": "oracle/ppo.c (Jacobi SVDs), GEMMs on OpenBLAS", "extrapolated": False, "seconds": sec}
        U, S, V = ppo.tsvdq(a, q, k)
        ppo.relative_error(a, ppo.tsvdq_reconstruct(U, S, V, q))
        sec = time.perf_counter() - t0
        return (8.0 * s1 * s2 * n3) / sec / 1e9, {
            "sample": f"oracle data Q + tsvdq + RE on a {s1}x{s2}x{n3} cut (p={p}, k={k})",
            "how": "oracle/ppo.c (Jacobi SVDs), GEMMs on OpenBLAS", "extrapolated": False, "seconds": sec}


class TsvdqSharded:
    """cfg5 pixel-sharded over the torchrun ranks (paper_2409_19402_b200/dist.py):
    every rank holds one lateral block; Gram partials -> pairwise tree across
    ranks (bitwise the 1-GPU Gram) -> replicated eigensolve -> local forward
    transform -> all_to_all reshard -> slice SVDs -> factor all-gather ->
    local fused residual -> all-reduce. Strong scaling (total work fixed)."""

    metric, unit = "tsvdq_input_GBps", "GB/s"

    def __init__(self, world, rank, local, n1=2048, n2=2048, n3=1024, p=128, k=32, seed=0):
        import torch
        from paper_2409_19402_b200 import dist as pdist, synth
        self.name = "cfg5"
        self.torch = torch
        self.dims = (n1, n2, n3, p, k)
        self.world = world
        self.be = pdist.DeviceBackend(f"cuda:{local}")
        self.plan = pdist.make_plan(n1, n2, n3, p, world, rank, self.be)
        self.pdist = pdist
        self.A = synth.cp_block_device(n1, n2, n3, self.plan.j0, self.plan.nj, 50, 1e-3, seed,
                                       device=f"cuda:{local}")
        self.in_bytes = 8.0 * n1 * n2 * n3  # the whole tensor (all ranks)
        self.re = None

    def config(self):
        n1, n2, n3, p, k = self.dims
        return {"workload": "cfg5 rank-50 CP + N(0,1e-3^2) noise tSVDQ with data-driven Q, pixel-sharded",
                "shape": [n1, n2, n3], "p": p, "k": k, "l2": "input > L2",
                "step": "dist.sharded_compress (Gram tree + NCCL all_gather / all_to_all / all_reduce)"}

    def step(self, L):
        _, _, _, _, k = self.dims
        self.be.L.ppc_set_stream(C.c_void_p(self.torch.cuda.current_stream().cuda_stream))
        *_, self.re = self.pdist.sharded_compress(self.A, self.plan, k, self.be)

    def value(self, sec):
        return self.in_bytes / sec / 1e9 / self.world  # main() multiplies by world

    def dominant(self, stages):
        return ("ozaki_syrk", "int8") if "ozaki_syrk" in stages else ("gram_syrk", "tensor")

    def e2e_setup(self):
        self.hA = flat_host(self.A)
        n1, n2, n3, p, k = self.dims
        self.h2d = 8 * n1 * n2 * n3
        self.d2h = 8 * (n3 * p + (n1 + n2 + 1) * k * p)

    def e2e_step(self, L):
        torch = self.torch
        n1, n2, n3, p, k = self.dims
        blk = self.torch.empty_like(self.A.permute(2, 1, 0)).reshape(-1)
        blk.copy_(self.hA, non_blocking=True)
        A = blk.view(n3, self.plan.nj, n1).permute(2, 1, 0)
        Q, U, S, V, _ = self.pdist.sharded_compress(A, self.plan, k, self.be)
        for t in (Q, U, S, V):
            t.cpu()

    def cpu_sample(self, ppo, threads):
        return Tsvdq.cpu_sample(self, ppo, threads)


class StarQSharded:
    """cfg4 row-sharded over the torchrun ranks (dist.sharded_star_q): rank r
    holds A's row block and B's lateral block, transforms both, all-gathers B^
    in slice groups overlapped with the facewise GEMMs, and inverse-transforms
    its own C rows. Strong scaling (the cfg4 product is fixed)."""

    name = "cfg4"
    metric, unit = "starq_tflops", "TFLOP/s"

    def __init__(self, world, rank, local, n1=1024, m=512, n2=1024, n3=256, p=64, seed=0):
        import torch
        import paper_2409_19402_b200 as pp
        from paper_2409_19402_b200 import dist as pdist, synth
        self.torch = torch
        self.pdist = pdist
        self.dims = (n1, m, n2, n3, p)
        self.world = world
        dev = f"cuda:{local}"
        self.be = pdist.DeviceBackend(dev)
        self.plan = pdist.make_star_plan(n1, m, n2, n3, p, world, rank)
        pl = self.plan
        A = synth.gaussian_device(n1, m, n3, seed, 1, device=dev)   # same bits as the 1-GPU run
        B = synth.gaussian_device(m, n2, n3, seed, 2, device=dev)
        self.A = A[pl.i0:pl.i0 + pl.rows].permute(2, 1, 0).contiguous().permute(2, 1, 0)
        self.B = B[:, pl.j0:pl.j0 + pl.cols].permute(2, 1, 0).contiguous().permute(2, 1, 0)
        del A, B
        self.Q = pp.to_device(pp.Transform("dct", n3, p).q, device=dev)
        self.flops = 2.0 * p * (n1 * m * n3 + m * n2 * n3 + n1 * m * n2 + n1 * n2 * n3)

    def config(self):
        n1, m, n2, n3, p = self.dims
        return {"workload": "cfg4 star-Q product, output rows sharded", "A": [n1, m, n3], "B": [m, n2, n3],
                "p": p, "transform": "dct", "l2": "inputs (2 GiB) > L2; no flush needed",
                "step": "dist.sharded_star_q (local transforms, NCCL all_gather of B^ in 4 slice groups "
                        "overlapped with the facewise GEMMs, local inverse)"}

    def step(self, L):
        self.be.L.ppc_set_stream(C.c_void_p(self.torch.cuda.current_stream().cuda_stream))
        self.C = self.pdist.sharded_star_q(self.A, self.B, self.Q, self.plan, self.be)

    def value(self, sec):
        return self.flops / sec / 1e12 / self.world  # main() multiplies by world

    def dominant(self, stages):
        return ("ozaki_gemm", "int8") if "ozaki_gemm" in stages else ("facewise", "tensor")

    def e2e_setup(self):
        self.hA = flat_host(self.A)
        self.hB = flat_host(self.B)
        n1, m, n2, n3, p = self.dims
        self.h2d = 8 * (self.plan.rows * m * n3 + m * self.plan.cols * n3)
        self.d2h = 8 * self.plan.rows * n2 * n3

    def e2e_step(self, L):
        torch = self.torch
        A = torch.empty_like(self.A.permute(2, 1, 0)).reshape(-1)
        B = torch.empty_like(self.B.permute(2, 1, 0)).reshape(-1)
        A.copy_(self.hA, non_blocking=True)
        B.copy_(self.hB, non_blocking=True)
        Av = A.view(self.A.shape[::-1]).permute(2, 1, 0)
        Bv = B.view(self.B.shape[::-1]).permute(2, 1, 0)
        Cr = self.pdist.sharded_star_q(Av, Bv, self.Q, self.plan, self.be)
        Cr.cpu()

    def cpu_sample(self, ppo, threads):
        return StarQ.cpu_sample(self, ppo, threads)


def make_workload(name, world=1, rank=0, local=0):
    if name == "cfg5" and world > 1:
        return TsvdqSharded(world, rank, local)
    if name == "cfg4" and world > 1:
        return StarQSharded(world, rank, local)
    if name == "cfg4":
        return StarQ()
    dims = {"cfg5": (2048, 2048, 1024, 128, 32), "cfg3": (512, 512, 224, 32, 16),
            "cfg2": (240, 320, 200, 20, 10)}[name]
    return Tsvdq(name, *dims)


# --------------------------------------------------------------- reference arm
def _cpu_threads():
    return os.cpu_count() or 1


def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm on the host cores (the C++
    reference cannot be built here: Eigen is absent), one bounded sample of
    the workload per step, all host threads: cfg5 on the LAPACK restatement
    (oracle/baseline.py, extrapolated from a pixel sample and whole slices),
    cfg4 the whole product on the C oracle with OpenBLAS GEMMs."""
    if rank != 0:
        return
    from oracle import ppo
    threads = _cpu_threads()
    ppo.use_openblas(threads=threads)
    ppo.set_threads(1 if args.workload == "cfg4" else threads)  # as cpu_leg

    class _Shim:  # cpu_sample needs only dims/name
        pass

    shim = _Shim()
    if args.workload == "cfg4":
        shim.dims, shim.name = (1024, 512, 1024, 256, 64), "cfg4"
        sample_fn, metric, unit = StarQ.cpu_sample, StarQ.metric, StarQ.unit
    else:
        shim.name, shim.dims = args.workload, TSVDQ_DIMS[args.workload]
        sample_fn, metric, unit = Tsvdq.cpu_sample, Tsvdq.metric, Tsvdq.unit
    for _ in range(min(args.warmup, 1) if args.workload in ("cfg4", "cfg5") else 0):
        sample_fn(shim, ppo, threads)
    vals, info = [], {}
    for _ in range(args.steps):
        v, info = sample_fn(shim, ppo, threads)
        vals.append(v)
    vals.sort()
    v = vals[len(vals) // 2]
    cpu = {"value": v, "unit": unit, "cores": threads, "kind": "port", "sample": info["sample"],
           "how": info["how"], "extrapolated": info["extrapolated"]}
    if args.workload == "cfg4":
        n1, m, n2, n3, p = shim.dims
        work = 2.0 * p * (n1 * m * n3 + m * n2 * n3 + n1 * m * n2 + n1 * n2 * n3) / 1e12
    else:
        n1, n2, n3 = shim.dims[:3]
        work = 8.0 * n1 * n2 * n3 / 1e9
    line = {"impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * work / v,  # of the whole workload (extrapolated from the sample where it says so)
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "sample": info["sample"]},
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


TSVDQ_DIMS = {"cfg5": (2048, 2048, 1024, 128, 32), "cfg3": (512, 512, 224, 32, 16),
              "cfg2": (240, 320, 200, 20, 10)}


# --------------------------------------------------------------------- legs
def roofline(wl, stages, peaks, workload, ms, bound_override=None):
    """Dominant kernel: algorithmic flops (or bytes) per launch / its average
    CUDA-event duration on the launching stream."""
    dom, bound = wl.dominant(stages)
    if bound_override:
        dom, bound = bound_override
    st = stages.get(dom, {"ms": float("nan"), "n": 1, "flops": 0.0, "bytes": 0.0})
    avg_ms = st["ms"] / max(1, st["n"])
    traffic, tsrc = ncu_traffic(workload, dom)
    if bound == "int8":
        achieved = (st["flops"] / max(1, st["n"])) / (avg_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["int8_tops"],
                "unit": "TFLOP/s", "op_kind": "int8 ops (TOPS) of the Ozaki digit products, tcgen05 kind::i8",
                "frac": achieved / peaks["int8_tops"], "traffic": traffic,
                "algorithmic_bytes": st["bytes"] / max(1, st["n"]), "kernel": dom,
                "peak_source": peaks["int8_src"], "traffic_source": tsrc,
                "frac_vs_int8_burst": (achieved / peaks["int8_burst_tops"]) if peaks.get("int8_burst_tops")
                else None,
                "frac_vs_cublaslt_int8": (achieved / peaks["int8_cublaslt_tops"]) if peaks["int8_cublaslt_tops"]
                else None,
                # the FP64 flops the digit products stand for: 21 digit pairs
                # (6-digit splits) or 28 (the 7-digit forward transform)
                "fp64_equivalent_tflops": achieved / (28.0 if dom == "ozaki_fwd" else 21.0)}
    elif bound == "tensor":
        achieved = (st["flops"] / max(1, st["n"])) / (avg_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"], "traffic": traffic,
                "algorithmic_bytes": st["bytes"] / max(1, st["n"]),
                "kernel": dom, "peak_source": peaks["fp64_src"] + " (FP64 DMMA; no tcgen05 f64 kind)",
                "traffic_source": tsrc}
    else:
        achieved = (st["bytes"] / max(1, st["n"])) / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "kernel": dom,
                "peak_source": peaks["hbm_src"], "traffic_source": tsrc}
    roof["ms_per_launch"] = avg_ms
    roof["share_of_step"] = st["ms"] / ms if ms > 0 else None
    return roof


def stage_summary(stages, ms):
    out = {}
    for name, s in stages.items():
        a_ms = s["ms"] / max(1, s["n"])
        out[name] = {"ms_per_launch": round(a_ms, 4), "launches": s["n"],
                     "share": round(s["ms"] / ms, 4) if ms > 0 else None}
        if s["flops"]:
            out[name]["tflops"] = round(s["flops"] / s["n"] / (a_ms / 1e3) / 1e12, 3)
        if s["bytes"]:
            out[name]["gbs"] = round(s["bytes"] / s["n"] / (a_ms / 1e3) / 1e9, 1)
    return out


def timed_leg(wl, L, stream, steps, warmup, dist_on):
    """W untimed steps, then K steps between CUDA events on the engine's
    stream with a barrier + synchronize on both sides; max over ranks."""
    import torch
    for _ in range(warmup):
        wl.step(L)
    sync_all(dist_on)
    L.ppc_launch_count(1)
    timing_report(L, reset=True)
    L.ppc_timing_enable(1)
    sync_all(dist_on)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        wl.step(L)
    e1.record(stream)
    sync_all(dist_on)
    L.ppc_timing_enable(0)
    ms = max_over_ranks(e0.elapsed_time(e1), dist_on)
    launches = int(L.ppc_launch_count(1))
    stages = timing_report(L, reset=True)
    return ms / steps, stages, launches


def e2e_leg(wl, L, steps, world, dist_on):
    import torch
    wl.e2e_setup()
    wl.e2e_step(L)  # warm
    sync_all(dist_on)
    t0 = time.perf_counter()
    for _ in range(steps):
        wl.e2e_step(L)
    torch.cuda.synchronize()
    sec = max_over_ranks((time.perf_counter() - t0) / steps, dist_on)
    return {"value": wl.value(sec) * world, "unit": wl.unit, "h2d_bytes_per_step": wl.h2d,
            "d2h_bytes_per_step": wl.d2h, "ms_per_step": sec * 1e3}


def cpu_leg(wl):
    try:
        from oracle import ppo
        threads = _cpu_threads()
        ppo.use_openblas(threads=threads)
        # star-Q: every host thread inside each BLAS GEMM (faster here than a
        # threaded slice loop over single-threaded GEMMs); tSVDQ: the slice
        # loop on every thread (the oracle's Jacobi SVDs do not use BLAS)
        ppo.set_threads(1 if wl.metric == StarQ.metric else threads)
        v, info = wl.cpu_sample(ppo, threads)
        return {"value": v, "unit": wl.unit, "cores": threads, "kind": "port", "sample": info["sample"],
                "how": info["how"], "extrapolated": info["extrapolated"], "cpu_seconds_per_step": info["seconds"],
                **({"parts": info["parts"]} if "parts" in info else {})}
    except Exception as ex:  # pragma: no cover
        return {"value": None, "unit": wl.unit, "cores": 0, "kind": "port", "sample": f"failed: {ex}"}


def golden_re():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "cfg5_dmma.json")) as f:
            return json.load(f)
    except Exception:
        return None


ARITHMETIC = ("FP64 emulated on the INT8 tensor cores (Ozaki digit splitting, exact int32 digit products, "
              "FP64 accumulation): 6-digit / 21-pair Gram SYRKs, 7-digit / 28-pair forward transform, "
              "3-6-level slice-SVD filter products; every other product (small GEMMs, polish, Rayleigh-Ritz, "
              "eigensolvers) on FP64 DMMA / FP64 FMA. value_fp64_dmma: the same step with every product on "
              "FP64 DMMA (ppc_set_ozaki(0))")


def spawn_ranks(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (one per GPU)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=os.environ.get("PPC_BENCH_WORKLOAD", "cfg5"),
                    choices=["cfg5", "cfg4", "cfg3", "cfg2"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the all-FP64-DMMA leg (cfg5)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg4 star-Q leg of the cfg5 run")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N-rank path on a one-GPU box: every rank on
    # cuda:0, collectives over gloo (NCCL refuses two ranks on one device);
    # the numbers of such a run are not a measurement
    shared_gpu = os.environ.get("PPC_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    dist_on = world > 1
    torch.cuda.set_device(local)
    if dist_on:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2409_19402_b200 as pp  # noqa: F401
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    if L.ppc_set_device(local):
        raise RuntimeError(L.ppc_last_error().decode())
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    L.ppc_set_stream(C.c_void_p(stream.cuda_stream))

    peaks = load_peaks()
    wl = make_workload(args.workload, world, rank, local)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        wl.step(L)
    sync_all(dist_on)
    clocks.mark()
    ms_step, stages, launches = timed_leg(wl, L, stream, args.steps, 0, dist_on)
    clk = clocks.stop()
    value = wl.value(ms_step / 1e3) * world  # whole job (sharded: value() divides by world)
    roof = roofline(wl, stages, peaks, args.workload, ms_step * args.steps)
    # the step's largest share may be latency-bound work with no throughput
    # roofline (the Householder reductions of the eigensolvers)
    tri = stages.get("eig.tridiag")
    if tri and tri["ms"] > stages.get(roof["kernel"], {"ms": 0.0})["ms"]:
        roof["largest_stage"] = {"stage": "eig.tridiag (sytrd_kernel)", "share": tri["ms"] / (ms_step * args.steps),
                                 "bound": "latency: grid barriers + L2 exchanges per column block"}
    re_main = getattr(wl, "re", None)

    e2e = None if args.no_e2e else e2e_leg(wl, L, args.steps, world, dist_on)

    # tSVDQ with a given Q (both timings): the Q of the last step
    given_q = None
    if hasattr(wl, "step_given_q") and args.workload in ("cfg5", "cfg3") and not args.no_fp64:
        full_step = wl.step
        wl.step = wl.step_given_q
        try:
            msq, stq, _ = timed_leg(wl, L, stream, args.steps, 1, dist_on)
        finally:
            wl.step = full_step
        given_q = {"value": wl.value(msq / 1e3) * world, "unit": wl.unit, "ms_per_step": msq, "steps": args.steps,
                   "warmup": 1, "step": "ppc_tsvdq(A, Q, k) = A x3 Q^T + facewise truncated SVDs "
                                        "(decompositions.cpp:62-83), Q given (device-resident, from the last "
                                        "compress step); the forward transform runs on FP64 DMMA here (no kept "
                                        "Gram digits to reuse)",
                   "stages": stage_summary(stq, msq * args.steps)}

    # the same step with every product on FP64 DMMA (no INT8 emulation)
    fp64 = None
    if args.workload == "cfg5" and not args.no_fp64:
        L.ppc_trim_workspace()
        assert L.ppc_set_ozaki(0) == 0
        try:
            k64 = max(2, min(3, args.steps))
            ms64, st64, _ = timed_leg(wl, L, stream, k64, 1, dist_on)
            roof64 = roofline(wl, st64, peaks, args.workload, ms64 * k64, bound_override=("gram_syrk", "tensor"))
            fp64 = {"value": wl.value(ms64 / 1e3) * world, "unit": wl.unit, "ms_per_step": ms64, "steps": k64,
                    "warmup": 1, "roofline": roof64, "relative_error": getattr(wl, "re", None),
                    "stages": stage_summary(st64, ms64 * k64)}
        finally:
            L.ppc_set_ozaki(1)
            L.ppc_trim_workspace()

    # the other half of the BASELINE metric: star-Q product TFLOP/s (cfg4)
    secondary = None
    if args.workload == "cfg5" and not args.no_secondary:
        wl4 = make_workload("cfg4", world, rank, local)
        ms4, st4, l4 = timed_leg(wl4, L, stream, args.steps, args.warmup, dist_on)
        secondary = {"metric": wl4.metric, "value": wl4.value(ms4 / 1e3) * world, "unit": wl4.unit,
                     "ms_per_step": ms4, "steps": args.steps, "warmup": args.warmup,
                     "config": wl4.config(), "gpu_launches": l4,
                     "roofline": roofline(wl4, st4, peaks, "cfg4", ms4 * args.steps),
                     "e2e": None if args.no_e2e else e2e_leg(wl4, L, args.steps, world, dist_on),
                     "stages": stage_summary(st4, ms4 * args.steps)}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            secondary["cpu_baseline"] = cpu_leg(wl4)
        del wl4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_leg(wl)

    if rank == 0:
        cfg = wl.config()
        sharded = isinstance(wl, (TsvdqSharded, StarQSharded))
        cfg["parallelism"] = (f"{'row' if isinstance(wl, StarQSharded) else 'pixel'}-sharded dp{world}" if sharded else
                              (f"replicas{world}" if world > 1 else "single"))
        if dist_on:
            cfg["comm"] = ({"backend": "gloo", "note": "PPC_BENCH_SHARED_GPU: all ranks on cuda:0, a functional "
                                                   "check of the N-rank path, not a measurement"}
                           if shared_gpu else
                           {"backend": "nccl", "nccl": ".".join(map(str, torch.cuda.nccl.version()))})
        line = {"metric": wl.metric, "value": value, "unit": wl.unit, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
                "dtype": "f64", "arithmetic": ARITHMETIC if args.workload != "cfg4" else
                ARITHMETIC.replace("6-digit / 21-pair Gram SYRKs, 7-digit / 28-pair forward transform, "
                                   "3-6-level slice-SVD filter products", "6-digit facewise product (rows "
                                   "passing the dynamic-range gate); transforms on FP64 DMMA"),
                "data": "synthetic", "config": cfg, "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "stages": stage_summary(stages, ms_step * args.steps)}
        if given_q is not None:
            line["value_given_q"] = given_q
        if fp64 is not None:
            line["value_fp64_dmma"] = fp64
        if secondary is not None:
            line["secondary"] = secondary
        if re_main is not None:
            rc = {"relative_error": re_main}
            if fp64 is not None and fp64["relative_error"] is not None:
                r64 = fp64["relative_error"]
                rc.update({"relative_error_fp64_dmma": r64, "rel_diff_vs_fp64_dmma": abs(re_main - r64) / r64})
            gold = golden_re() if args.workload == "cfg5" and not sharded else None
            if gold:
                rl = gold["relative_error_lapack"]
                rc.update({"relative_error_lapack_golden": rl, "rel_diff_vs_lapack_golden": abs(re_main - rl) / rl,
                           "golden": "tests/golden/cfg5_dmma.json (tools/golden_cfg5.py)"})
            diffs = [v for kk, v in rc.items() if kk.startswith("rel_diff")]
            if diffs:
                rc["ok_1e-10"] = all(d <= 1e-10 for d in diffs)
            line["result_check"] = rc
        print(json.dumps(line), flush=True)

    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
