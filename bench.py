#!/usr/bin/env python
"""bench.py -- equilibration throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config.workload): BASELINE.json configs[2] ("c3"): sparse CSR A,
m = 2e6, n = 1e6, Zipf(1.5) row lengths on [1, 1e4] (nnz = 1.535e8), entries
N(0,1) with row/column scalings exp(N(0,1.5)); auto targets, T = 100
stochastic iterations, seed 0.  It is the config BASELINE's metric is quoted on
at 1/2/4/8 GPUs.  A "step" is one complete sgd_equilibrate call: all T*(n+m)
probe signs generated on device, T fused SGD passes over CSR(A) and CSR(A^T),
final exp.  value = whole-job iterations per second (strong scaling: the same
matrix is row-sharded over N GPUs).

Our arm prints one JSON line with value (matrix resident in HBM), e2e (one-shot
C-ABI call from pinned host CSR: upload + device transpose + T iterations +
download), roofline (live CUDA-event time of the fused iteration kernel), the
CPU baseline (oracle C port, single thread, bounded sample), clocks and the
number of our kernels launched.  --impl reference times the reference's own
sources (oracle/_ref, built from /root/reference against eigen-lite) on the
host: rank 0 only, single thread (the reference has no threading).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "equilibration iters/sec and achieved HBM GB/s (fraction of 8 TB/s) at 1/2/4/8 B200"
UNIT = "iterations/s"
CONFIG_ID = 3
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c4 LSQR and c2 dense keys")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for the timing barriers (gloo + "
                         "EQUIL_HOST_EXCHANGE=2 + --device 0: several ranks on one GPU, "
                         "a test of the N > 1 path)")
    ap.add_argument("--device", type=int, default=-1, help="GPU of every rank (default LOCAL_RANK)")
    ap.add_argument("--ref-iters", type=int, default=3,
                    help="reference arm: SGD iterations per step (one sgd_equilibrate call)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def algorithmic_bytes(inst) -> float:
    """Bytes one SGD iteration must move:
    A and A^T values + int32 columns (24 B/nnz), both row pointers, the two
    gathered vectors once, u/ubar/v/vbar read+write, next e.*s / d.*w written,
    the sign bits."""
    m, n, nnz = inst.m, inst.n, inst.nnz
    return 24.0 * nnz + 52.125 * (m + n) + 8.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """DRAM bytes per SGD iteration (both SGD kernel launches) from the
    committed ncu --set full capture (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["sgd_iter_kernel"]["dram_bytes_per_launch"])
    except Exception:
        return None


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def workload_config(inst, world: int) -> dict:
    """config dict shared by both arms (the driver compares them)."""
    return {"workload": "c3: sparse CSR 2e6 x 1e6, Zipf(1.5) rows on [1,1e4], "
                        "exp(N(0,1.5)) scalings, T=100, seed 0, auto targets",
            "m": inst.m, "n": inst.n, "nnz": inst.nnz, "iterations_per_step": inst.iterations,
            "l2": "inputs larger than L2 (CSR(A)+CSR(A^T) = 3.7 GB >> 126 MB)",
            "parallelism": f"rows of A and A^T sharded over {world} GPU(s)"}


def host_cpu() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


FIXTURE = os.path.join(ROOT, "tests", "golden", "fullsize_c3.json")


def sha(a) -> str:
    import hashlib

    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check_vs_fixture(inst, vecs: dict) -> dict:
    """Compare u, v, d, e of the benched run (c3, T=100, seed 0) with the digest
    the oracle and the reference's own sources produced (tests/golden/
    make_fullsize.py); the matrix digest proves it is the same instance."""
    try:
        with open(FIXTURE) as f:
            fx = json.load(f)
    except OSError:
        return {"bit_identical_to_oracle": None, "why": "fixture missing"}
    want = fx["instance"]
    same_inst = (sha(inst.row_ptr), sha(inst.col), sha(inst.val)) == (
        want["row_ptr"], want["col"], want["val"])
    ok = same_inst and inst.iterations == fx["config"]["iterations"] and all(
        sha(vecs[k]) == fx["result"][k] for k in "uvde")
    return {"bit_identical_to_oracle": bool(ok), "fixture": "tests/golden/fullsize_c3.json",
            "same_instance": bool(same_inst)}


def lsqr_bytes(inst) -> float:
    """Bytes one LSQR iteration must move: A and A^T once
    (24 B/nnz), row pointers, m-side u, d, b read + d.u gathered + u written,
    n-side v, e, x, w read + e.v, e.x gathered + v, x, w written."""
    m, n, nnz = inst.m, inst.n, inst.nnz
    return 24.0 * nnz + 4.0 * (m + n) + 8.0 * (5 * m + 9 * n)


def c4_cpu_lsqr(inst, b) -> dict:
    """The reference's LSQR per iteration on the host: the oracle
    C port (bit-identical to the reference's sources), 1 thread, on the full c3
    matrix; the difference of a 3- and a 1-iteration solve."""
    import oracle
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    O = oracle.c_oracle()
    t0 = time.perf_counter()
    O.lsqr(A, b, 1, 0.0)
    t1 = time.perf_counter()
    O.lsqr(A, b, 3, 0.0)
    t2 = time.perf_counter()
    per = ((t2 - t1) - (t1 - t0)) / 2
    return {"ms_per_lsqr_iteration": per * 1e3, "cores": 1, "kind": "port",
            "sample": "oracle lsqr on the full c3 matrix, 3 minus 1 iterations, 1 thread",
            **host_cpu()}


def c4_experiment(eq, M, inst, peak: float, curve_every: int = 25, cpu: bool = False) -> dict:
    """BASELINE configs[3] on the resident c3 matrix: plain lsqr (500) and
    lsqr_preconditioned (T=50 + 500), tol 0 -- run_lsqr_experiment's two
    variants (src/experiments.cpp:234-281).  Per-iteration time from the
    difference of a 500- and a 0-iteration solve; residual curves sampled every
    `curve_every` iterations; every history entry and x checked against the
    fixtures tests/golden/fullsize_c4{p,q}.json."""
    from paper_1602_06621_b200 import configs
    b = configs.rhs(inst)
    iters, T = 500, 50
    pe = eq.EquilibrationParams(iterations=T, seed=0)
    eq.lsqr(M, b, 2, 0.0)  # warm
    t0 = time.perf_counter()
    eq.lsqr(M, b, 0, 0.0)
    t_zero = time.perf_counter() - t0
    t0 = time.perf_counter()
    plain = eq.lsqr(M, b, iters, 0.0)
    t_plain = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = eq.lsqr_preconditioned(M, b, pe, iters, 0.0)
    t_pre = time.perf_counter() - t0
    per_it = (t_plain - t_zero) / iters
    B = lsqr_bytes(inst)
    check = {}
    for tag, run in (("c4p", plain), ("c4q", pre)):
        try:
            with open(os.path.join(ROOT, "tests", "golden", f"fullsize_{tag}.json")) as f:
                fx = json.load(f)["result"]
            hist = [float.fromhex(x) for x in fx["residual_history"]]
            check[tag] = bool(list(run.residual_history) == hist and sha(run.x) == fx["x"])
        except OSError:
            check[tag] = None

    def curve(h, offset=0):
        return {str(k): h[k] for k in range(0, len(h), curve_every)} | {str(len(h) - 1): h[-1]}

    return {"workload": "c4: c3's A, b = A x_true + 0.01 N(0,1); plain lsqr 500 iterations and "
                        "lsqr_preconditioned T=50 + 500, tol 0",
            "ms_per_lsqr_iteration": per_it * 1e3,
            "lsqr_s": {"plain": t_plain, "preconditioned": t_pre, "zero_iterations": t_zero},
            "roofline": {"bound": "hbm", "bytes_per_iteration": B,
                         "achieved": B / per_it / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B / per_it / 1e9 / peak},
            "residual_vs_total_iteration": {"plain": curve(list(plain.residual_history)),
                                            f"equil{T}": curve(list(pre.residual_history))},
            "check": {"bit_identical_to_oracle": check},
            "cpu_baseline": c4_cpu_lsqr(inst, b) if cpu else None}


def c2_dense(eq, peak: float) -> dict:
    """BASELINE configs[1]: dense 4096 x 2048, T=100, seed 1 (matrix resident)."""
    from paper_1602_06621_b200 import configs
    inst = configs.config(2)
    D = eq.ExplicitMatrix.dense(inst.dense)
    p = eq.EquilibrationParams(iterations=inst.iterations, seed=inst.seed)
    ms = []
    for _ in range(5):
        eq.sgd_equilibrate(D, p)
        ms.append(eq.last_loop_ms(D)[0])
    D.close()
    per = statistics.median(ms[1:]) / 1e3 / inst.iterations
    B = 8.0 * inst.m * inst.n + 48.125 * (inst.m + inst.n)
    return {"workload": "c2: dense 4096 x 2048 fp64 row-major, T=100, seed 1",
            "us_per_iteration": per * 1e6, "iterations_per_s": 1.0 / per,
            "roofline": {"bound": "hbm", "bytes_per_iteration": B, "achieved": B / per / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": B / per / 1e9 / peak,
                         "note": "single-pass bytes; A (67 MB) is L2-resident across iterations"}}


def cpu_baseline(inst, iters: int):
    import numpy as np  # noqa: F401
    import oracle
    A = oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val)
    O = oracle.c_oracle()
    t0 = time.perf_counter()
    O.sgd_equilibrate(A, alpha=inst.alpha, beta=inst.beta, iterations=iters, seed=inst.seed)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{iters} SGD iterations of the full c3 matrix (oracle/equil_oracle.c, "
                      f"bit-identical to the reference's sources), 1 thread, {dt:.2f} s",
            **host_cpu()}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1602_06621_b200 as eq
    from paper_1602_06621_b200 import configs

    rank, world, local = dist_env()
    if args.gpus != world and world == 1 and args.gpus > 1:
        raise SystemExit("run N>1 under torch.distributed.run (one process per GPU)")
    if args.device >= 0:
        local = args.device
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64,
                         device=torch.device("cuda", local) if args.dist_backend == "nccl"
                         else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    inst = configs.config(CONFIG_ID)
    T = inst.iterations
    nccl_id = None
    if world > 1:
        obj = [eq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    M = eq.ExplicitMatrix.from_csr(inst.m, inst.n, inst.row_ptr, inst.col, inst.val,
                                   device=local, rank=rank, world_size=world, nccl_id=nccl_id)
    p = eq.EquilibrationParams(alpha=inst.alpha, beta=inst.beta, iterations=T, seed=inst.seed)
    dev = torch.device("cuda", local)
    u = torch.empty(inst.m, dtype=torch.float64, device=dev)
    v = torch.empty(inst.n, dtype=torch.float64, device=dev)
    d = torch.empty(inst.m, dtype=torch.float64, device=dev)
    e = torch.empty(inst.n, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(eq._lib.load().equil_matrix_stream(M._h))

    def step():
        return eq.sgd_equilibrate_device(M, p, u.data_ptr(), v.data_ptr(), d.data_ptr(),
                                         e.data_ptr())

    for _ in range(args.warmup):
        res = step()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    barrier()
    clocks.start()
    l0 = eq.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    loop_ms = []
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
        loop_ms.append(eq.last_loop_ms(M)[0])
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    launches = eq.kernel_launches() - l0
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        elapsed = max_over_ranks(elapsed)
    value = T * args.steps / elapsed

    # ---- roofline of the dominant kernel (fused SGD pass), live CUDA events
    B = algorithmic_bytes(inst)
    kern_s = max(statistics.mean(loop_ms), 1e-9) / 1e3 / T  # per launch (T launches)
    per_gpu_bytes = B / world
    achieved = per_gpu_bytes / kern_s / 1e9
    peak, peak_src = peaks()
    traffic = ncu_traffic()

    # ---- e2e at N > 1 (the one-GPU e2e runs after the extras, once the resident handle is closed)
    e2e = None
    if world > 1:
        # the same public path at N GPUs: every rank builds its shard from the
        # pinned host CSR (handle + communicator), runs T iterations and reads
        # the gathered u, v, d, e back to the host; max over ranks
        pin_rp = torch.from_numpy(inst.row_ptr).pin_memory()
        pin_c = torch.from_numpy(inst.col).pin_memory()
        pin_v = torch.from_numpy(inst.val).pin_memory()
        ts = []
        r = None
        for _ in range(min(args.e2e_steps, 3)):  # (each one builds a communicator)
            obj = [eq.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            barrier()
            t0 = time.perf_counter()
            M2 = eq.ExplicitMatrix.from_csr(inst.m, inst.n, pin_rp.numpy(), pin_c.numpy(),
                                            pin_v.numpy(), device=local, rank=rank,
                                            world_size=world, nccl_id=obj[0])
            r = eq.sgd_equilibrate(M2, p)
            M2.close()
            ts.append(max_over_ranks(time.perf_counter() - t0))
        e2e_s = statistics.mean(ts)
        h2d = int(inst.row_ptr.nbytes + inst.col.nbytes + inst.val.nbytes) * world
        d2h = int(8 * 2 * (inst.m + inst.n)) * world
        e2e = {"value": T / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "s_per_step": e2e_s,
               "samples_s": [round(t, 4) for t in ts],
               "path": "ExplicitMatrix.from_csr on every rank (upload, device transpose, "
                       "shard, communicator) + sgd_equilibrate to host"}
        if rank == 0:  # the sharded result must equal one GPU's bit for bit
            one = eq.sgd_equilibrate_csr(inst.m, inst.n, pin_rp.numpy(), pin_c.numpy(),
                                         pin_v.numpy(), p, device=local)
            check = {"bit_identical_to_1gpu": bool(
                all(np.array_equal(getattr(r, k), getattr(one, k)) for k in "uvde"))}
        barrier()
        del r

    extra = {}
    if world == 1:
        # the benched result (device buffers of the last timed step) and the e2e
        # result, against the oracle / reference digest of this exact run
        vecs = {k: t.cpu().numpy() for k, t in zip("uvde", (u, v, d, e))}
        check = check_vs_fixture(inst, vecs)
        if not args.no_extras:
            extra["c4_lsqr"] = c4_experiment(eq, M, inst, peak,
                                             cpu=rank == 0 and not args.no_cpu_baseline)
            extra["c2_dense"] = c2_dense(eq, peak)

    # ---- e2e through the one-shot C ABI from pinned host memory.  The resident
    # handle is closed first: a second live handle of this size on the device makes
    # about one one-shot call in ten stall (tools/pool_probe.py), and a caller of the
    # one-shot entry point has none.
    exchange = eq.exchange_mode(M)
    sweep = eq.sweep_active(M)
    if world == 1:
        M.close()
        pin_rp = torch.from_numpy(inst.row_ptr).pin_memory()
        pin_c = torch.from_numpy(inst.col).pin_memory()
        pin_v = torch.from_numpy(inst.val).pin_memory()
        # pinned result buffers: the device->host read of u, v, d, e is inside the step
        pin_out = tuple(torch.empty(k, dtype=torch.float64).pin_memory().numpy()
                        for k in (inst.m, inst.n, inst.m, inst.n))
        for _ in range(3):  # warm (module load, jump polys, pool growth, pinned mappings)
            eq.sgd_equilibrate_csr(inst.m, inst.n, pin_rp.numpy(), pin_c.numpy(), pin_v.numpy(),
                                   p, device=local, out=pin_out)
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            r = eq.sgd_equilibrate_csr(inst.m, inst.n, pin_rp.numpy(), pin_c.numpy(),
                                       pin_v.numpy(), p, device=local, out=pin_out)
            ts.append(time.perf_counter() - t0)
        e2e_s = statistics.mean(ts)  # (every sample and the median are reported beside it)
        h2d = int(inst.row_ptr.nbytes + inst.col.nbytes + inst.val.nbytes)
        d2h = int(8 * 2 * (inst.m + inst.n))
        e2e = {"value": T / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "s_per_step": e2e_s,
               "s_per_step_median": statistics.median(ts),
               "samples_s": [round(t, 4) for t in ts],
               "path": "equil_sgd_equilibrate_csr (pinned host CSR in, pinned u, v, d, e out: "
                       "upload, device transpose, T iterations, download)"}
        del r
        check["e2e_bit_identical_to_oracle"] = check_vs_fixture(
            inst, dict(zip("uvde", pin_out)))["bit_identical_to_oracle"]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(inst, args.cpu_iters)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator restating BASELINE configs[2])",
            "config": workload_config(inst, world),
            "ms_per_iteration": elapsed / args.steps / T * 1e3,
            # a step = sign stream (K1, all T iterations) + init + the T-iteration
            # loop + final exp (signs reported apart, and inside value)
            "step_breakdown_ms": {"loop": kern_s * 1e3 * T,
                                  "signs_init_final": elapsed / args.steps * 1e3 - kern_s * 1e3 * T},
            "achieved_GBps": B * value / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("sweep_kernel + sell_warp_kernel + sgd_update_rows_kernel: "
                                    "one iteration = A's rows of > 512 entries on the column "
                                    "sweep (xs in shared-memory panels), every other row of A "
                                    "and A^T on interleaved warp slices, then the u/v update "
                                    "of every row") if sweep else
                                   ("sell_warp_kernel + sell_long_kernel + "
                                    "sgd_update_rows_kernel: one iteration = A and A^T passes "
                                    "over interleaved row slices (warp slices and "
                                    "warp-specialised long-row CTAs, concurrent), then the u/v "
                                    "update of every row"),
                         "long_rows": "column sweep" if sweep else "long-slice kernel",
                         "bytes_per_launch": per_gpu_bytes, "launch_ms": kern_s * 1e3,
                         "peak_source": peak_src},
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
            "flags": {"box_feasible": res.box_feasible, "iterate_bound_ok": res.iterate_bound_ok},
            "exchange": exchange, "check": check, **extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def load_instance_without_repo_libs(tmp: str):
    """c3 generated in a CHILD process (which loads the repo's generator
    library) and read back here from raw files, so the reference process maps
    no repo shared object -- only oracle/_ref/libequil_ref.so."""
    import numpy as np
    code = ("import sys, numpy as np; sys.path.insert(0, %r); "
            "from paper_1602_06621_b200 import configs; i = configs.config(%d); "
            "[np.save(%r + '/' + k + '.npy', getattr(i, k)) for k in ('row_ptr', 'col', 'val')]; "
            "print(i.m, i.n, i.iterations, i.seed, i.alpha, i.beta)") % (ROOT, CONFIG_ID, tmp)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True)
    m, n, T, seed, alpha, beta = out.stdout.split()

    class Inst:
        pass
    inst = Inst()
    inst.m, inst.n, inst.iterations, inst.seed = int(m), int(n), int(T), int(seed)
    inst.alpha, inst.beta = float(alpha), float(beta)
    for k in ("row_ptr", "col", "val"):
        setattr(inst, k, np.load(os.path.join(tmp, k + ".npy")))
    inst.nnz = int(inst.row_ptr[-1])
    return inst


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    if not os.path.exists(oracle.REF_PATH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libequil_ref.so was "
                          "not built (needs /root/reference at build time)"}))
        return
    with tempfile.TemporaryDirectory() as tmp:
        inst = load_instance_without_repo_libs(tmp)
    R = oracle.ref_oracle()
    t0 = time.perf_counter()
    RM = R.matrix(oracle.CsrArrays(inst.m, inst.n, inst.row_ptr, inst.col, inst.val))
    build_s = time.perf_counter() - t0
    T = max(1, args.ref_iters)  # SGD iterations of the full matrix per step (bounded sample)
    for _ in range(args.warmup):
        RM.sgd_equilibrate(alpha=inst.alpha, beta=inst.beta, iterations=T, seed=inst.seed)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        RM.sgd_equilibrate(alpha=inst.alpha, beta=inst.beta, iterations=T, seed=inst.seed)
    dt = time.perf_counter() - t0
    value = T * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3 * inst.iterations / T,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator restating BASELINE configs[2])",
        "config": workload_config(inst, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"sgd_equilibrate with T={T} per call on the full c3 matrix "
                                   f"({args.steps} timed calls; ms_per_step scaled to T="
                                   f"{inst.iterations}); the reference's sources (oracle/_ref) "
                                   "on eigen-lite, 1 thread (the reference has no threading; "
                                   f"ExplicitMatrix::sparse build {build_s:.1f} s untimed)",
                         **host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
