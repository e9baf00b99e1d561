#!/usr/bin/env python
"""bench.py -- IBF-MAT apply throughput on B200 (BASELINE.json metric:
"BF apply N.RHS/s and % of HBM/FP32 roofline at N=2^20, 256 RHS").

One step = one bf_apply of the whole hot path (S0, all transfer levels with the
switch, SL) over one batch of 256 complex64 RHS of BASELINE config 4 (N = 2^20,
leaf 64, r = 10, 2 amplitude terms), inputs resident in HBM.  Multi-GPU: one
process per GPU (torchrun; `--gpus N` without torchrun launches it), RHS-sharded
as config 4 says: rank q applies the replicated plan to columns
[q 256/N, (q+1) 256/N) of the one seeded batch, no collective on the data path
(strong scaling; value = N.256 / max-over-ranks time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  See DESIGN.md section 7 for every field.
"""
from __future__ import annotations

import argparse
import ctypes
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

from paper_1803_04128_b200 import workloads as W  # noqa: E402

METRIC = "BF apply N·RHS/s and % of HBM/FP32 roofline at N=2^20, 256 RHS"
UNIT = "N*RHS/s"
# FP32 SIMT peak from the unit counts and max clock: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


L2_BYTES = 126 << 20   # B200 L2

def _peaks():
    """HBM GB/s and the TF32 tensor peak (TFLOP/s) with their sources.  TF32 = the measured sustained cuBLAS
    bf16 rate x the guide's nominal tf32/bf16 ratio (1.1 / 2.25): the kernels run inside a ~100 ms step under
    the power cap (B200_PROFILING.md)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        hbm, src = float(p["hbm_gbs"]), "measured"
        bf16 = float(p.get("bf16_tflops_sustained", p["bf16_tflops"]))
        tsrc = "MEASURED_PEAKS.json bf16_tflops_sustained x 1.1/2.25 (nominal tf32/bf16)"
    except Exception:
        hbm, src = 6650.0, "fallback"
        bf16, tsrc = 1400.0, "fallback sustained bf16 1.4 PF x 1.1/2.25"
    return hbm, src, bf16 * 1.1 / 2.25, tsrc


def _sustained():
    """Measured sustained device rates (tools/sustained_peaks.py: >= 4 s FFMA and kind::tf32 MMA loads on every SM,
    under the power cap) from the newest committed capture, or None."""
    for rnd in ("r2",):
        try:
            with open(os.path.join(ROOT, "profiles", f"{rnd}_sustained_peaks.json")) as f:
                return json.load(f)
        except Exception:
            continue
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


def _ncu_traffic(workload, cls):
    """DRAM bytes per launch of kernel class `cls` from the newest committed ncu capture of this workload
    (profiles/r2_traffic_<workload>.json, else r1_), or None."""
    for rnd in ("r2", "r1"):
        try:
            with open(os.path.join(ROOT, "profiles", f"{rnd}_traffic_{workload}.json")) as f:
                return json.load(f)["bytes_per_launch"].get(cls)
        except Exception:
            continue
    return None


def stage_model(w, nvec, info):
    """Algorithmic flops and bytes per launch of each kernel class.
    Transfer classes: a launch performs class_levels/class_launches fused levels; each launch reads and
    writes the coefficient array once.  The switch is folded into the level-h blocks at plan finalization,
    so it adds no work of its own."""
    N, n0, r, na, nrhs = w.n, w.leaf, w.rank, w.n_amp, nvec // w.n_amp
    c = 8  # bytes per complex64
    if info.get("structured") and not info["tc_classes"]:
        # structured factors: per (pair, vector) a phase cmul (6 flops) per input element and a
        # real x complex MAC (4 flops) per Lagrange weight; one level per launch; level h dense (16 r^2)
        io = c * 2 * N * r * nvec
        return {
            "s0": (N * nvec * (6 * n0 + 4 * r * n0) + 6 * N * nvec,
                   c * (N * nrhs + na * N + N * n0 + N * r * nvec)),
            "xfer_first_half": (N * nvec * (12 * r + 8 * r * r), io + c * N * 2 * r),
            "xfer_switch": (16 * N * r * r * nvec, io + c * N * 2 * r * r),
            "xfer_second_half": (N * nvec * (8 * r * r + 16 * r), io + c * N * 2 * r),
            "sl": (N * nvec * n0 * (4 * r + 8) + 8 * N * nvec, c * (N * r * nvec + N * n0 + na * N + N * nrhs)),
        }
    out = {
        "s0": (8 * N * n0 * r * nvec + 6 * N * nvec, c * (N * nrhs + na * N + N * n0 * r + N * r * nvec)),
        "sl": (8 * N * n0 * r * nvec + 8 * N * nvec, c * (N * r * nvec + N * n0 * r + na * N + N * nrhs)),
    }
    for k in ("xfer_first_half", "xfer_switch", "xfer_second_half"):
        n, lv = info["class_launches"][k], info["class_levels"][k]
        if n == 0:
            out[k] = (0, 0)
            continue
        flops = lv * 16 * N * r * r * nvec / n
        byts = c * (2 * N * r * nvec) + c * lv * 2 * N * r * r / n
        out[k] = (flops, byts)
    return out


def rhs_columns(nrhs: int, world: int, rank: int):
    """Columns [c0, c1) of the global RHS batch that rank `rank` of `world` applies (contiguous,
    balanced; the RHS are independent units, so the ranks' results concatenate to the 1-GPU result)."""
    return rank * nrhs // world, (rank + 1) * nrhs // world


def _self_launch(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: start N ranks on this node with torch.distributed.run (127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpu_oracle_sample(w, g0=None, adjoint=False):
    """The oracle as it stands on the host cores: the config's full-N butterfly for ONE RHS column (its n_amp
    vectors), blocks generated on the fly in FP64 -- timed -- and, untimed, the accuracy triplet of that column
    on the eps^b row sample: oracle BF vs the direct sum (eps^b), the GPU column g0 vs the direct
    sum, and the GPU column vs the oracle BF on all N rows (the parity quantity, bar 1e-5)."""
    import oracle
    F = W.rhs(w.n, w.nrhs, w.seed, cols=[0])
    bf_apply = oracle.bf_apply_adjoint if adjoint else oracle.bf_apply
    direct = oracle.direct_adjoint_rows if adjoint else oracle.direct_rows
    t0 = time.perf_counter()
    gb = bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    dt = time.perf_counter() - t0
    out = {"value": w.n * 1 / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "seconds": dt,
           "sample": f"{w.name} at full N=2^{w.log2n}, 1 of {w.nrhs} RHS columns ({w.n_amp} amplitude vectors), "
                     f"FP64 oracle {'ADJOINT (O8) ' if adjoint else ''}incl. on-the-fly block generation; "
                     f"metric scaled per N*RHS"}
    if g0 is not None:
        rows = W.sample_rows(w.n, w.seed)
        t1 = time.perf_counter()
        gd = direct(w.kernel, w.amp, w.log2n, F, rows)[:, 0]
        dt_direct = time.perf_counter() - t1
        # the other oracle leg SURVEY 8(d) names: the direct O(N^2) sum, timed on its 256-row sample (one row of one
        # column = one N*RHS unit)
        out["legs"] = {"bf_otf_incl_block_generation": {"value": out["value"], "seconds": dt},
                       "direct_sum_row_sample": {"value": len(rows) / dt_direct, "seconds": dt_direct,
                                                 "rows": len(rows)}}
        out["accuracy"] = {"column": 0, "rows": len(rows), "eps": w.eps,
                           "eps_b_oracle_bf_vs_direct": float(oracle.rel_l2(gb[rows, 0], gd)),
                           "gpu_vs_direct": float(oracle.rel_l2(g0[rows].astype(np.complex128), gd)),
                           "gpu_vs_oracle_bf_all_rows": float(oracle.rel_l2(g0.astype(np.complex128), gb[:, 0]))}
    return out


def run_reference(args, w, rank, world):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    F = W.rhs(w.n, w.nrhs, w.seed, cols=[0])
    for _ in range(args.warmup):
        oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    dt = (time.perf_counter() - t0) / args.steps
    val = w.n / dt
    sample = (f"each step: cfg4 at full N=2^{w.log2n}, 1 of {w.nrhs} RHS columns (2 amplitude vectors), "
              f"FP64 CPU oracle with on-the-fly blocks")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Gaussian RHS, closed-form kernel)",
        "config": {"workload": "cfg4", "n": w.n, "leaf": w.leaf, "rank": w.rank, "n_amp": w.n_amp,
                   "nrhs_per_step": 1},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_nufft(args, w, rank, world, local):
    """--path nufft: the NUFFT path (include/bf_nufft.h) on the config's workload, RHS-sharded like the butterfly.
    Roofline: the whole apply (place + cuFFT + interpolation) against HBM, algorithmic bytes = F and G once plus
    the fine grids' M placed frequencies written once, the grids read and written once by the FFT and read once
    by the interpolation (3.5 x 8 n_sub nv n_f)."""
    import torch
    import torch.distributed as dist
    from paper_1803_04128_b200 import bf

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c0, c1 = rhs_columns(w.nrhs, world, rank)
    nloc = c1 - c0
    chunk = args.chunk or nloc
    t0 = time.perf_counter()
    plan = bf.NufftPlan.build_fio(bf.fio_of(w), device=local, max_nrhs_chunk=chunk, eps=w.eps)
    t_build = time.perf_counter() - t0
    info = plan.info()
    F = W.rhs(w.n, w.nrhs, w.seed) if world == 1 else W.rhs(w.n, w.nrhs, w.seed, cols=range(c0, c1))
    Fd = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gd = torch.empty_like(Fd)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        plan.apply(Fd, Gd, nloc, stream=stream)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            plan.apply(Fd, Gd, nloc, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    hbm, hbm_src, _, _ = _peaks()
    nv = min(chunk, nloc) * w.n_amp
    grid_bytes = 8 * 2 * nv * info["grid"] * (-(-nloc // chunk))
    byts = 16 * w.n * nloc + 3.5 * grid_bytes + 8 * 2 * w.n_amp * w.n
    roof = {"bound": "hbm", "achieved": byts / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})", "traffic": None,
            "kernel": "whole apply: place_kernel + cuFFT C2C (library) + interp_kernel",
            "algorithmic_bytes": byts}
    roof["frac"] = roof["achieved"] / roof["peak"]
    acc = cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        rows = W.sample_rows(w.n, w.seed)
        F0 = W.rhs(w.n, w.nrhs, w.seed, cols=[0])
        ts = time.perf_counter()
        gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F0, rows)[:, 0]
        dt = time.perf_counter() - ts
        g0 = Gd[0].cpu().numpy().astype(np.complex128)
        acc = {"column": 0, "rows": len(rows), "gpu_vs_direct": float(oracle.rel_l2(g0[rows], gd)),
               "eps": w.eps, "width": info["width"]}
        cpu = {"value": len(rows) / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
               "seconds": dt, "sample": f"{w.name}: {len(rows)} rows of RHS column 0 by the direct sum O0 (FP64; "
                                        "the oracle evaluates eqn:tg3 by its definition), one row = one N*RHS unit"}
    if rank == 0:
        out = {"metric": METRIC, "value": w.n * w.nrhs / (ms / 1e3), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "impl": "nufft-path",
               "dtype": "c64 (fp32 place/interp, cuFFT C2C single precision)",
               "data": "synthetic (seeded Gaussian complex64 RHS; closed-form FIO kernel)",
               "config": {"workload": f"{w.name}-nufft", "n": w.n, "n_amp": w.n_amp, "nrhs_per_gpu": nloc,
                          "global_batch": w.nrhs, "max_nrhs_chunk": chunk, "width": info["width"],
                          "grid": info["grid"], "submatrices": 2,
                          "parallelism": f"rhs-sharded x{world} (no collective)",
                          "l2": f"no flush: the fine grids ({grid_bytes / 1e9:.3g} GB) exceed the 126 MB L2"},
               "roofline": roof, "e2e": None, "gpu_launches": info["launches_per_chunk"] * (-(-nloc // chunk))
               * args.steps, "cpu_baseline": cpu, "clocks": clk.summary(), "accuracy": acc,
               "plan_build_s": t_build}
        print(json.dumps(out), flush=True)
    plan.destroy()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--nrhs", type=int, default=None, help="global RHS batch (default: the config's), split over the ranks")
    ap.add_argument("--chunk", type=int, default=None, help="max_nrhs_chunk (default: all RHS in one chunk)")
    ap.add_argument("--log2n", type=int, default=None, help="override N (profiling of a smaller instance only)")
    ap.add_argument("--index-shard", action="store_true",
                    help="split ONE batch by index over the ranks (NCCL all-to-all at level h; cfg5's mode)")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="one CUDA-graph launch per step (bf_apply_graph); auto: for steps of <= 2^22 N*vectors")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", choices=["copy", "fused"], default="copy",
                    help="index-shard exchange: NCCL send/recv step, or peer stores from the level-h launch")
    ap.add_argument("--host-pieces", type=int, default=None,
                    help="bf_apply_host pipeline pieces per chunk (BF_OPT_HOST_PIECES; e2e only)")
    ap.add_argument("--no-leaf-multicast", action="store_true",
                    help="TF32 SL without the 2-CTA cluster Ux multicast (BF_OPT_LEAF_MULTICAST = 0)")
    ap.add_argument("--no-tc", action="store_true", help="every stage on the FP32 kernels (BF_OPT_TENSOR_CORES = 0)")
    ap.add_argument("--no-small-batch", action="store_true",
                    help="small vector batches: one transfer level per launch (BF_OPT_SMALL_BATCH = 0)")
    ap.add_argument("--band-compose", type=int, default=None, choices=[0, 1],
                    help="tensor-core band: composed two-level operator (1) or level by level (0) (BF_OPT_BAND_COMPOSE)")
    ap.add_argument("--structured", action="store_true",
                    help="structured interpolative factors: phases + shared Lagrange matrices (NEXT-1)")
    ap.add_argument("--factors", choices=["auto", "interpolative", "structured", "recompressed"], default="auto",
                    help="factor form: auto = per config (DESIGN.md 7): cfg3/cfg4 recompressed 12 -> 8, cfg2/cfg5 "
                         "structured, cfg1 interpolative")
    ap.add_argument("--recompress", type=int, default=None, metavar="RP",
                    help="recompress the interpolative factorization of rank --build-rank to rank RP (NEXT-3)")
    ap.add_argument("--build-rank", type=int, default=12, help="interpolative rank before --recompress")
    ap.add_argument("--path", choices=["bf", "nufft"], default="bf",
                    help="bf: the IBF-MAT butterfly (the north_star path); nufft: the NUFFT path of the unified "
                         "framework (eqn:tg3 with type-2 NUFFTs on the xi<0 / xi>=0 submatrices, DESIGN.md 5.8)")
    ap.add_argument("--adjoint", action="store_true",
                    help="time the adjoint apply K* (bf_plan_create_adjoint from the forward plan)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and "WORLD_SIZE" in os.environ and args.gpus != 1:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    # Host OpenMP threads (the untimed factor builder; the oracle of the reference arm).  torchrun exports
    # OMP_NUM_THREADS=1 to every rank by default, which would make the builder and the reference arm
    # single-threaded: replace that default.  GPU arm: share the node's cores between its ranks; reference
    # arm: rank 0 works alone and takes all of them.  Set before our libraries load libgomp, and also
    # through omp_set_num_threads in case it is already initialized.
    torchrun_default = os.environ.get("OMP_NUM_THREADS") == "1" and "TORCHELASTIC_RUN_ID" in os.environ
    if torchrun_default or (local_world > 1 and "OMP_NUM_THREADS" not in os.environ):
        ncores = os.cpu_count() or 1
        nthr = ncores if args.impl == "reference" else max(1, ncores // local_world)
        os.environ["OMP_NUM_THREADS"] = str(nthr)
        try:
            ctypes.CDLL("libgomp.so.1").omp_set_num_threads(ctypes.c_int(nthr))
        except OSError:
            pass
    w = W.CONFIGS[args.config]
    if args.nrhs:
        w = w.with_(nrhs=args.nrhs)
    if args.log2n:
        w = w.with_(log2n=args.log2n)

    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    if args.path == "nufft":
        run_nufft(args, w, rank, world, local)
        return
    # factor form: the fastest measured form of each config at the config's accuracy
    if args.factors == "auto" and not (args.structured or args.recompress or args.adjoint or args.index_shard):
        args.factors = {"cfg3": "recompressed", "cfg4": "recompressed", "cfg2": "structured",
                        "cfg5": "structured"}.get(args.config, "interpolative")
    if args.factors == "recompressed" and not args.recompress:
        args.recompress = 8
    if args.factors == "structured":
        args.structured = True

    import torch
    import torch.distributed as dist
    from paper_1803_04128_b200 import bf

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    if args.index_shard:
        c0, c1 = 0, w.nrhs   # every rank holds all columns, a 1/G slice of the rows
    else:
        c0, c1 = rhs_columns(w.nrhs, world, rank)
    nloc = c1 - c0   # columns this rank applies per step
    chunk = args.chunk or nloc
    t0 = time.perf_counter()
    if args.index_shard:
        # one batch split by index: rank q owns xi-rows and x-rows [q N/G, (q+1) N/G) (strong scaling)
        obj = [bf.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        plan = bf.Plan.build_fio_sharded(bf.fio_of(w), rank, world, obj[0], device=local, max_nrhs_chunk=chunk)
        if args.exchange == "fused":
            plan.set_option(bf.BF_OPT_EXCHANGE, 1)   # collective: every rank
        F = W.rhs(w.n, w.nrhs, w.seed)
        rows = w.n // world
        F = np.asfortranarray(F[rank * rows:(rank + 1) * rows])
    else:
        if args.adjoint:
            # the forward plan only lends its compact factors (chunk 1: no workspace to speak of, no tensor-core
            # images); the adjoint plan re-assembles them on the device, then the forward is released
            fwd = bf.Plan.build_fio(bf.fio_of(w), device=local, max_nrhs_chunk=1)
            plan = fwd.adjoint(chunk)
            fwd.destroy()
        elif args.recompress:
            # the interpolative factorization at --build-rank (chunk 1: no workspace, no tensor-core images), its
            # balanced truncation to rank RP on the device, then the source is released
            src = bf.Plan.build_fio(bf.fio(w.kernel, w.amp, w.log2n, w.log2leaf, args.build_rank), device=local,
                                    max_nrhs_chunk=1)
            plan = src.recompress(args.recompress, chunk)
            src.destroy()
            w = w.with_(rank=args.recompress)
        elif args.structured:
            plan = bf.Plan.build_fio_structured(bf.fio_of(w), device=local, max_nrhs_chunk=chunk)
        else:
            plan = bf.Plan.build_fio(bf.fio_of(w), device=local, max_nrhs_chunk=chunk)
        # this rank's RHS: columns [c0, c1) of the one seeded global batch (strong scaling)
        F = W.rhs(w.n, w.nrhs, w.seed) if world == 1 else W.rhs(w.n, w.nrhs, w.seed, cols=range(c0, c1))
    t_build = time.perf_counter() - t0
    if args.no_tc:
        plan.set_tensor_cores(False)
    if args.no_small_batch:
        plan.set_option(bf.BF_OPT_SMALL_BATCH, 0)
    if args.band_compose is not None:
        plan.set_option(bf.BF_OPT_BAND_COMPOSE, args.band_compose)
    if args.no_leaf_multicast:
        plan.set_option(bf.BF_OPT_LEAF_MULTICAST, 0)
    if args.host_pieces:
        plan.set_option(bf.BF_OPT_HOST_PIECES, args.host_pieces)
    info = plan.info()
    Fd = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gd = torch.empty_like(Fd)
    stream = torch.cuda.current_stream()

    # launch: one CUDA-graph launch per step (bf_apply_graph) where the step's kernels run for microseconds and
    # the host launch rate would bound it, else the eager stream launches of bf_apply
    use_graph = args.graph == "on" or (args.graph == "auto" and not args.index_shard
                                       and w.n * nloc * w.n_amp <= (1 << 22))
    if use_graph and args.index_shard:
        raise SystemExit("--graph on: bf_apply_graph does not take NCCL index-sharded plans")

    def step():
        (plan.apply_graph if use_graph else plan.apply)(Fd, Gd, nloc, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # L2: a working set that fits the 126 MB L2 would stay resident between steps, so those configs flush it
    # (a 256 MB write between steps, outside the timed spans) and time every step alone
    work_bytes = 2 * 8 * w.n * nloc + 8 * (w.n >> ((world.bit_length() - 1) if args.index_shard else 0)) * w.rank * min(chunk, nloc) * w.n_amp + info["factor_bytes"]
    flush = work_bytes < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device="cuda") if flush else None

    # ---- timed region: K steps, device-timed with CUDA events on the launching stream ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        if flush:
            spans = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(args.steps)]
            for i, (a, b) in enumerate(spans):
                scratch.fill_(i & 0xFF)
                a.record(stream)
                step()
                b.record(stream)
        else:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = (sum(a.elapsed_time(b) for a, b in spans) if flush else ev0.elapsed_time(ev1)) / args.steps
    del scratch
    # per-kernel times: the same K steps again with the library's CUDA events around every launch (a separate
    # pass, so the events' own cost stays out of ms_per_step; for the millisecond-scale steps the two agree)
    plan.set_timing(True)
    for _ in range(args.steps):
        plan.apply(Fd, Gd, nloc, stream)
    torch.cuda.synchronize()
    ktimes = plan.timing()
    ms_timed_pass = sum(v[0] for v in ktimes.values()) / args.steps
    plan.set_timing(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    chunks = -(-nloc // chunk)
    launches = info["launches_per_chunk"] * chunks * args.steps
    value = w.n * w.nrhs / (ms / 1e3)   # the whole batch of w.nrhs columns per step, all ranks together

    # ---- roofline of the dominant kernel class ----
    hbm, hbm_src, tf32, tf32_src = _peaks()
    wl = w.with_(log2n=w.log2n - (world.bit_length() - 1)) if args.index_shard else w   # this rank's share
    model = stage_model(wl, min(chunk, nloc) * w.n_amp, info)
    # the level-h exchange moves (G-1)/G of the local coefficients out and as much in
    model["exchange"] = (0, 2 * 8 * wl.n * w.rank * min(chunk, nloc) * w.n_amp * (world - 1) // world)
    tc_classes = set(info["tc_classes"])

    def tpeak(k):
        return tf32

    def times(k):
        """(compute seconds, hbm seconds) of one launch of class k at its peaks.  Tensor-core classes
        issue 3 split products per FP32-accurate product (3xTF32)."""
        f, b = model[k]
        tcomp = 3 * f / (tpeak(k) * 1e12) if k in tc_classes else f / (FP32_PEAK_TFLOPS * 1e12)
        return tcomp, b / (hbm * 1e9)

    dom = max((k for k in ktimes if k != "exchange"), key=lambda k: ktimes[k][0])   # largest share of the step
    dms, dn = ktimes[dom]
    flops, byts = model[dom]
    avg_s = dms / dn / 1e3
    t_comp, t_hbm = times(dom)
    if t_hbm >= t_comp:
        roof = {"bound": "hbm", "achieved": byts / avg_s / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})"}
    elif dom in tc_classes:
        roof = {"bound": "tensor", "achieved": 3 * flops / avg_s / 1e12, "peak": tpeak(dom), "unit": "TFLOP/s",
                "peak_source": tf32_src
                + "; achieved counts the 3 split passes of each algorithmic FP32 flop"}
    else:
        roof = {"bound": "alu", "achieved": flops / avg_s / 1e12, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "peak_source": "FP32 FFMA from unit counts: 148 SM x 128 lanes x 2 x 1.965 GHz (DESIGN.md 5)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    sus = _sustained()
    if sus and roof["bound"] in ("tensor", "alu"):
        # the same achieved rate against the rate a seconds-long load of that unit sustains on this pool's B200s
        key = "tf32_tflops_sustained" if roof["bound"] == "tensor" else "ffma_tflops_sustained"
        roof["peak_sustained_measured"] = sus[key]
        roof["frac_of_sustained_measured"] = roof["achieved"] / sus[key]
        roof["sustained_source"] = "profiles/r2_sustained_peaks.json (tools/sustained_peaks.cu)"
    wname = (args.config + ("-adjoint" if args.adjoint else "") + ("-structured" if args.structured else "")
             + (f"-recompressed-r{args.build_rank}to{args.recompress}" if args.recompress else ""))
    roof["traffic"] = _ncu_traffic(wname if not (args.log2n or args.adjoint or args.nrhs or args.chunk) else None, dom)
    roof["kernel"] = dom
    roof["tensor_cores"] = dom in tc_classes
    roof["avg_launch_ms"] = avg_s * 1e3
    roof["share_of_step"] = dms / (ms_timed_pass * args.steps)
    # whole-step roofline fractions (level-by-level and fused), DESIGN.md section 5
    tot_f = sum(model[k][0] * ktimes[k][1] for k in model) / args.steps
    lbl = sum(max(times(k)) * ktimes[k][1] for k in model if k != "exchange") / args.steps
    comp = sum(times(k)[0] * ktimes[k][1] for k in model if k != "exchange") / args.steps
    fused = max(comp, (16 * wl.n * nloc + info["factor_bytes"]) / (hbm * 1e9))

    # ---- end to end: host buffers through the C ABI, copies inside the timed region ----
    # e2e: K steps of bf_apply_host_async (each step copies its F host->device, applies, copies G device->host;
    # consecutive steps overlap one step's copies with the neighbours' applies), then bf_apply_host_wait: the
    # last G is on the host when the clock stops.  e2e_sync: bf_apply_host, which returns with G on the host.
    e2e = e2e_sync = None
    if not args.no_e2e:
        Fh = torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory()
        Gh = torch.empty_like(Fh).pin_memory()
        nb = Fd.numel() * 8

        def maxrank(x):
            if world > 1:
                t = torch.tensor([x], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                x = float(t.item())
            return x

        plan.apply_host_async(Fh, Gh, nloc, stream)   # warm-up (allocates the staging slots once)
        plan.apply_host_wait()
        ne = max(2, args.steps)
        barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            plan.apply_host_async(Fh, Gh, nloc, stream)
        plan.apply_host_wait()
        te = maxrank((time.perf_counter() - t0) / ne)
        e2e = {"value": w.n * w.nrhs / te, "unit": UNIT, "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
               "ms_per_step": te * 1e3, "steps": ne, "api": "bf_apply_host_async x K, then bf_apply_host_wait"}
        plan.apply_host(Fh, Gh, nloc, stream)         # warm-up of the synchronous path's staging
        ns = max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(ns):
            plan.apply_host(Fh, Gh, nloc, stream)     # synchronizes: the result is on the host
        ts = maxrank((time.perf_counter() - t0) / ns)
        e2e_sync = {"value": w.n * w.nrhs / ts, "unit": UNIT, "ms_per_step": ts * 1e3, "steps": ns,
                    "api": "bf_apply_host (returns with G on the host)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        g0 = None if args.index_shard else Gd[0].cpu().numpy()   # column 0 of the last timed apply
        cpu = cpu_oracle_sample(W.CONFIGS[args.config].with_(nrhs=w.nrhs, log2n=w.log2n) if args.recompress else w,
                                g0, adjoint=args.adjoint)
        if args.recompress and cpu.get("accuracy"):
            # the oracle BF is the rank-r interpolative one: a different (equally accurate) operator than the
            # recompressed one -- the comparison that matters is the GPU against the direct sum
            cpu["accuracy"]["note"] = (f"GPU runs the rank-{args.build_rank} factorization recompressed to rank "
                                       f"{args.recompress}; gpu_vs_oracle_bf compares two different "
                                       f"approximations of the same kernel, gpu_vs_direct is the accuracy")

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": ("c64: tcgen05 split products with FP32 accumulation (" +
                      ", ".join(f"{k} 3xTF32" for k in sorted(tc_classes)) + ")")
                     if tc_classes else "c64 (fp32 FFMA)",
            "data": "synthetic (seeded Gaussian complex64 RHS; closed-form FIO kernel; factors from the host builder)",
            "config": {"workload": wname, "n": w.n, "leaf": w.leaf, "rank": w.rank, "n_amp": w.n_amp,
                       "nrhs_per_gpu": nloc, "global_batch": w.nrhs, "max_nrhs_chunk": chunk,
                       "parallelism": (f"index-sharded x{world} (level-h exchange: "
                                       + ("peer stores from the level-h launch)" if args.exchange == "fused"
                                          else "NCCL all-to-all)") if args.index_shard
                                       else f"rhs-sharded x{world}: rank q applies columns [q {w.nrhs}/{world}, "
                                            f"(q+1) {w.nrhs}/{world}) (no collective)"),
                       "l2": ((f"flushed: the working set ({work_bytes / 1e6:.3g} MB) fits the 126 MB L2, so a "
                               f"{2 * L2_BYTES >> 20} MB buffer is written between steps and each step is timed "
                               "alone") if flush else
                              (f"no flush: the working set (F {8 * w.n * nloc / 1e9:.2g} GB, coefficients "
                               f"{8 * wl.n * w.rank * min(chunk, nloc) * w.n_amp / 1e9:.3g} GB per level, factors "
                               f"{info['factor_bytes'] / 1e9:.3g} GB) exceeds the 126 MB L2")),
                       "launch": ("one CUDA-graph launch per step (bf_apply_graph)" if use_graph
                                  else "stream launches (bf_apply)"),
                       "tensor_core_classes": info["tc_classes"], "tc_weight_bytes": info["tc_weight_bytes"],
                       "factor_bytes": info["factor_bytes"], "structured": bool(info["structured"])},
            "roofline": roof,
            "step_roofline": {"level_by_level_ms": lbl * 1e3, "fused_ms": fused * 1e3,
                              "frac_level_by_level": lbl * 1e3 / ms, "frac_fused": fused * 1e3 / ms,
                              "algorithmic_tflops": tot_f / (ms / 1e3) / 1e12},
            "kernels": {k: {"ms_total": v[0], "launches": v[1], "ms_avg": (v[0] / v[1] if v[1] else None),
                            "flops_per_launch": model[k][0], "bytes_per_launch": model[k][1]}
                        for k, v in ktimes.items()},
            "e2e": e2e, "e2e_sync": e2e_sync, "gpu_launches": launches, "cpu_baseline": cpu, "clocks": clk.summary(),
            "accuracy": cpu.pop("accuracy", None) if cpu else None,
            "plan_build_s": t_build, "kernel_sum_ms_per_step": ms_timed_pass,
        }
        print(json.dumps(out), flush=True)
    plan.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
