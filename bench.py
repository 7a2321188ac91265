#!/usr/bin/env python3
"""Benchmark of the APSP hot path (BASELINE.json metric) -- one JSON line on stdout.

Workload (N=1): blocked Floyd-Warshall, distances + predecessors, on the reference
generator graph GenParams(n=16384, rho=0.1, alpha=100, seed=7+n) as int32 -- the metric's
size ("APSP time and min-plus updates/sec (n^3/s) at n=16384").  A step is one complete
APSP solve of that matrix (input scan, tier conversion, all n/128 pivot rounds, certificate,
conversion back) with the input already resident in HBM.  N>1 (torchrun): each rank owns a
row band of a weak-scaled problem n(N) = 16384 * N^(1/3) (n^3 per GPU fixed) and the pivot
row panel is broadcast over NCCL each round (paper_2310_03983_b200.distributed).

value        = n^3 * steps / max-over-ranks device time                 [updates/s]
e2e          = same metric through the C-ABI host-buffer call apsp_solve_host (pinned
               host input -> device -> host dist + pred), copies inside the timed region
roofline     = the dominant kernel (min-plus tile kernel, FW phase 3): algorithmic updates
               per launch / its CUDA-event launch time, against the measured issue ceiling
               of its inner-loop instruction (profiles/r01_microbench_ops.txt)
cpu_baseline = the oracle port of reference fw_classic (C/OpenMP, int64, all host threads)
               on a bounded sample of k-steps of the same matrix
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "APSP time and min-plus updates/sec (n^3/s) at n=16384; % of FP32 CUDA-core peak"
UNIT = "updates/s"
FP32_CORE_PEAK = 148 * 128 * 1965e6 / 2          # 18.6 T upd/s at max clock
# Measured issue ceilings of the inner-loop instruction of each tier's phase-3 kernel
# (tools/microbench/ops.cu; profiles/r01_microbench_ops.txt; argmin_i32: profiles/r02_microbench_ops.txt)
TIER_PEAK = {"u8": 37.07e12, "u16": 37.07e12, "w32": 17.98e12, "i32": 6.12e12, "f32": 20.17e12, "i64": 6.05e12}
TIER_OP = {"u8": "VIADDMNMX.U16x2 (2 upd/instr)", "u16": "VIADDMNMX.U16x2 (2 upd/instr)",
           "w32": "VIADDMNMX.U32 (1 upd/instr)", "i32": "IADD/ISETP/IMNMX/SEL compare-select (argmin_i32)",
           "f32": "FADD2 + FMNMX3 (deferred argmin; the FMNMX3 ALU rate bounds it)", "i64": "compare-select int64"}
BLOCK = 0          # 0: the library's size-aware default (apsp_info.block reports it)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_input(n: int, rho: float, seed: int):
    from paper_2310_03983_b200 import GenParams, dense_costs

    t = time.perf_counter()
    h = dense_costs(GenParams(n, rho, 100, seed), np.int32)
    log(f"[bench] generated n={n} rho={rho} seed={seed} in {time.perf_counter() - t:.1f}s "
        f"(density {(h != 0x3FFFFFFF).sum() / (n * n):.4f})")
    return h


class CpuSampler:
    """Bounded sample of the oracle port of reference fw_classic on the bench matrix.

    FW's early k-steps are nearly free on a sparse input (rows with d[i][k] = INF are skipped,
    solvers.py:85-87), so the sample is taken at steady state: steps [0, k_warm) run once
    untimed, the state is saved, and each sample re-runs steps [k_warm, k_warm + K) from a
    copy of that state.  K is sized to ~budget_s of CPU time.
    """

    def __init__(self, h32: np.ndarray, budget_s: float, k_warm: int = 512):
        from oracle import oracle as orc

        self.orc = orc
        self.n = h32.shape[0]
        self.threads = orc.threads()
        h64 = h32.astype(np.int64)
        h64[h32 == 0x3FFFFFFF] = orc.INF_RAW
        self.k_warm = min(k_warm, self.n // 2)
        d, p = orc.fw_classic(h64, k_end=self.k_warm, nthreads=self.threads)
        self.d0, self.p0 = d, p
        del h64
        t = time.perf_counter()
        dd, pp = d.copy(), p.copy()
        copy_s = time.perf_counter() - t
        t = time.perf_counter()
        orc.fw_steps(dd, pp, self.k_warm, self.k_warm + 8, self.threads)
        one = (time.perf_counter() - t) / 8
        self.K = int(max(4, min(self.n - self.k_warm, budget_s / max(one, 1e-6))))
        self.copy_s = copy_s

    def run(self) -> float:
        dd, pp = self.d0.copy(), self.p0.copy()
        t = time.perf_counter()
        self.orc.fw_steps(dd, pp, self.k_warm, self.k_warm + self.K, self.threads)
        return time.perf_counter() - t

    def describe(self) -> str:
        return (f"oracle fw_classic (C/OpenMP int64, solvers.py:77-95) steady-state k-steps "
                f"{self.k_warm}..{self.k_warm + self.K} of n={self.n} ({self.K}*n^2 updates), resumed from "
                f"the saved state after {self.k_warm} untimed steps; {self.threads} threads. "
                f"Bias: a steady-state window runs slower than the whole-solve average (the early k-steps "
                f"skip rows with d[i][k] = INF): at n=16384 the full oracle solve took 333 s (13.2 G upd/s, "
                f"16 threads, profiles/r01_summary.md) against 12.1-12.6 G upd/s in this window, so the "
                f"sampled rate understates the CPU by ~5-9%")

    FULL_SOLVE = {"n": 16384, "s": 333.0, "rate": 16384 ** 3 / 333.0, "threads": 16,
                  "source": "profiles/r01_summary.md (full oracle fw_classic solve on the GPU box host)"}


def cpu_baseline(h32: np.ndarray, budget_s: float = 12.0) -> dict:
    s = CpuSampler(h32, budget_s)
    dt = s.run()
    rate = s.K * s.n * s.n / dt
    return {"value": rate, "unit": UNIT, "cores": s.threads, "kind": "port",
            "sample": s.describe() + f"; {dt:.1f}s; full solve extrapolates to {s.n ** 3 / rate:.0f}s",
            "full_solve_reference_point": CpuSampler.FULL_SOLVE}


def networkx_baseline(n: int = 1024, rho: float = 0.1) -> dict | None:
    """NetworkX floyd_warshall_numpy (float64, distances only, single thread), a full solve of
    GenParams(n, rho, 100, 7+n) -- the survey's third comparison point."""
    try:
        import networkx as nx
    except ImportError:
        return None
    from paper_2310_03983_b200 import GenParams, generate

    g = generate(GenParams(n, rho, 100, 7 + n))
    G = nx.DiGraph()
    G.add_nodes_from(range(n))
    G.add_weighted_edges_from(g.edges)
    t = time.perf_counter()
    nx.floyd_warshall_numpy(G)
    dt = time.perf_counter() - t
    rate = n ** 3 / dt
    return {"value": rate, "unit": UNIT, "cores": 1, "kind": "networkx",
            "sample": f"networkx {nx.__version__} floyd_warshall_numpy full solve n={n} rho={rho} ({dt:.2f}s, "
                      f"distances only); n=16384 extrapolates to {16384 ** 3 / rate / 3600:.1f} h"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    n = args.n or weak_n(ws)
    h = make_input(n, args.rho, 7 + n)
    s = CpuSampler(h, args.ref_step_s)
    for _ in range(args.warmup):
        s.run()
    dt = sum(s.run() for _ in range(args.steps))
    rate = args.steps * s.K * n * n / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": scaling_of(args), "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference generator)",
        "config": config(n, args.rho, ws),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": s.threads, "kind": "port",
                         "sample": "each step = " + s.describe(), "full_solve_reference_point": CpuSampler.FULL_SOLVE},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def scaling_of(args) -> str:
    return "strong" if args.strong else "weak"


def weak_n(ws: int) -> int:
    n = 16384 * ws ** (1.0 / 3.0)
    return int(round(n / (256 * ws)) * 256 * ws) if ws > 1 else 16384


def config(n, rho, ws):
    return {"workload": f"blocked Floyd-Warshall APSP, distances+predecessors, n={n}, generator graph "
                        f"GenParams(n, rho={rho}, alpha=100, seed=7+n), int32 in/out",
            "n": n, "rho": rho, "layout": "1D row bands" if ws > 1 else "single GPU",
            "parallelism": f"rowband{ws}" if ws > 1 else "1gpu",
            "l2": "inputs larger than L2 (1 GiB int32 dist + 1 GiB pred + 256 MiB u8 store per GPU)"}


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--gpus", type=int, default=1)
    ap_.add_argument("--steps", type=int, default=5)
    ap_.add_argument("--warmup", type=int, default=3)
    ap_.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap_.add_argument("--n", type=int, default=0)
    ap_.add_argument("--rho", type=float, default=0.1)
    ap_.add_argument("--no-cpu", action="store_true")
    ap_.add_argument("--no-e2e", action="store_true")
    ap_.add_argument("--no-tiers", action="store_true", help="skip the w32 / i32 / continuous-fp32 variants")
    ap_.add_argument("--ref-step-s", type=float, default=8.0)
    ap_.add_argument("--block", type=int, default=BLOCK, help="pivot block (multiple of 128; 0 = library default)")
    ap_.add_argument("--sharded", action="store_true", help="use the multi-GPU row-band path even at N=1")
    ap_.add_argument("--alg", default="fw", choices=["fw", "rkleene"],
                     help="multi-GPU leg: row-band FW (default) or replicated R-Kleene with row-band products")
    ap_.add_argument("--strong", action="store_true",
                     help="strong scaling (BASELINE C4): n=32768 at every N instead of the weak-scaled n(N)")
    args = ap_.parse_args()
    ws, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank per GPU")
    if args.strong and not args.n:
        args.n = 32768
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    if ws > 1 or args.sharded:
        from paper_2310_03983_b200 import distributed

        return distributed.bench_main(args, METRIC, UNIT, config, make_input, weak_n, ClockSampler,
                                      cpu_baseline=cpu_baseline, tier_peak=TIER_PEAK, tier_op=TIER_OP)
    return bench_single(args)


def spawn_ranks(n_gpus: int):
    """`bench.py --gpus N` outside torchrun: relaunch this command as N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1; fails loudly if fewer GPUs are visible."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but only {have} CUDA device(s) are visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    log("[bench] launching", " ".join(cmd))
    os.execvp(cmd[0], cmd)


def bench_single(args):
    import torch

    import paper_2310_03983_b200 as ap
    from paper_2310_03983_b200 import _native as nat

    n = args.n or 16384
    block = args.block
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = nat.load()
    h_np = make_input(n, args.rho, 7 + n)
    h = torch.from_numpy(h_np).to(dev)
    dist = torch.empty_like(h)
    pred = torch.empty((n, n), dtype=torch.int32, device=dev)
    wsb = max(lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, dt, n, block) for dt in (nat.DTYPE_I32, nat.DTYPE_F32))
    work = torch.empty(wsb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    info = nat.ApspInfo()

    def step():
        with torch.cuda.stream(stream):
            dist.copy_(h)
        st = lib.apsp_fw_blocked(nat.DTYPE_I32, n, dist.data_ptr(), n, pred.data_ptr(), n, block, nat.TIER_AUTO,
                                 work.data_ptr(), wsb, sp, ctypes.byref(info))
        nat.check(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness guard on the measured configuration: a cheap certificate on the result
    ok, why = ap.check_pred_tree(h, dist, pred, ap.INF32) if n <= 16384 else (True, "skipped")
    if not ok:
        raise SystemExit(f"bench result failed the predecessor certificate: {why}")
    tier = nat.TIER_NAMES[info.tier]
    launches_per_step = info.launches
    block = info.block or block
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = lib.apsp_launch_count()
    with ClockSampler(0) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    launches_timed = lib.apsp_launch_count() - launches0
    ms_step = total_ms / args.steps
    value = n ** 3 * args.steps / (total_ms / 1e3)

    # dominant kernel: FW phase-3 min-plus tile launches, timed with CUDA events on their stream
    # (apsp_set_profiling) in one extra, untimed solve without the lookahead stream, so no
    # phase-1/2 kernel shares the SMs with a phase-3 launch: the kernel's own rate.
    def profile():
        os.environ["APSP_NO_LOOKAHEAD"] = "1"
        try:
            lib.apsp_set_profiling(1)
            step()
            torch.cuda.synchronize()
            lib.apsp_set_profiling(0)
        finally:
            os.environ.pop("APSP_NO_LOOKAHEAD", None)
        return info.kernel_launches, info.kernel_ms

    N = (n + block - 1) // block * block
    # phase 3 of one pivot round updates every tile outside the pivot cross: (N-b)^2 * b
    # (3a + 3b launches together); a solve has N/b rounds
    upd_phase3 = (N // block) * (N - block) ** 2 * block
    kl, kms = profile()
    achieved = upd_phase3 / (kms / 1e3) if kl else None
    peak = TIER_PEAK.get(tier)
    kname = f"minplus_nt_kernel<{tier}> (FW phase 3, bulk-staged)" if tier in ("u8", "u16") else \
        f"minplus_{tier}_kernel (FW phase 3)"
    roofline = {"bound": "alu", "kernel": kname, "op": TIER_OP.get(tier),
                "achieved": achieved / 1e12 if achieved else None, "peak": peak / 1e12 if peak else None,
                "unit": "T updates/s", "frac": (achieved / peak) if achieved and peak else None,
                "traffic": None, "launches_per_step": kl, "kernel_ms_per_step": kms,
                "updates_per_step": upd_phase3,
                "measurement": "CUDA events around every phase-3 launch on its stream, one extra solve without the "
                               "lookahead stream (no concurrent kernels)",
                "step_frac": value / peak if peak else None,
                "peak_source": "measured issue ceiling of the inner-loop instruction, profiles/r01_microbench_ops.txt"}
    # DRAM traffic of one phase-3b launch from the committed ncu --set full capture of this
    # configuration (profiles/ncu_phase3b.json, tools/ncu_summary.py); null for other configs
    cap = Path(__file__).resolve().parent / "profiles" / "ncu_phase3b.json"
    if cap.exists() and tier == "u8" and n == 16384 and block == 1024:
        c = json.loads(cap.read_text())
        roofline["traffic"] = c["traffic_bytes"]
        roofline["traffic_launch"] = {"updates": c["updates"], "duration_ms_isolated": c["duration_ms"],
                                      "achieved_isolated": c["achieved_T"], "frac_isolated": c["frac_of_dpx_ceiling"],
                                      "source": "profiles/ncu_phase3b.json (ncu --set full of the 7th long phase-3b launch, round 2, tools/p3_capture.sh; summary profiles/r02_ncu_phase3b.txt)"}

    parity = reference_digest(dist, n, args.rho)
    tiers = None if args.no_tiers else bench_tiers(lib, nat, h, dist, pred, work, stream, n, args, block)

    e2e = api = None
    if not args.no_e2e:
        e2e = bench_e2e(lib, nat, h_np, n, args, block)
        api = bench_python_api(h_np, n)
    cpu = nxb = None
    if not args.no_cpu:
        cpu = cpu_baseline(h_np)
        nxb = networkx_baseline()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "apsp_time_s": ms_step / 1e3, "higher_is_better": True, "scaling": scaling_of(args),
        "vs_baseline": None, "dtype": f"int16x2 keys / uint8 store (tier {tier}); int32 in/out" if tier == "u8"
        else f"tier {tier}; int32 in/out",
        "data": "synthetic (reference generator, bit-identical to apsp.generate)",
        "config": config(n, args.rho, 1), "block": block,
        "pct_fp32_core_peak": value / FP32_CORE_PEAK,
        "fp32_core_peak": FP32_CORE_PEAK,
        "clocks": clk.summary(), "gpu_launches": launches_timed,
        "tier": tier, "max_finite_distance": info.max_finite,
        "roofline": roofline, "e2e": e2e, "python_api_e2e": api, "cpu_baseline": cpu, "networkx_baseline": nxb,
        "parity": parity, "tiers": tiers,
    }
    print(json.dumps(line), flush=True)


def reference_digest(dist, n, rho):
    """Untimed: sha256 of the device result in the reference's int64 form against the digest of
    the REFERENCE's own solve of this graph (tests/golden/large.json, make_golden_large.py)."""
    import hashlib

    import paper_2310_03983_b200 as ap

    gold = json.loads((ROOT / "tests" / "golden" / "large.json").read_text())
    ref = next((v for v in gold.values() if v["n"] == n and v["rho"] == rho and v["seed"] == 7 + n), None)
    if ref is None:
        return {"checked": False, "why": f"no reference digest recorded for n={n} rho={rho}"}
    d = dist.cpu().numpy()
    d64 = d.astype(np.int64)
    d64[d == ap.INF32] = ap.INF_RAW
    got = hashlib.sha256(np.ascontiguousarray(d64).tobytes()).hexdigest()
    if got != ref["dist_sha256"]:
        raise SystemExit(f"bench result differs from the reference's distances (sha256 {got} != {ref['dist_sha256']})")
    return {"checked": True, "dist_sha256_equals_reference": True,
            "reference": f"apsp {ref['algorithm']} on GenParams({n}, {rho}, 100, {7 + n}), int64, "
                         f"{ref['solve_s']} s on {ref['cores']} cores (tests/golden/large.json)",
            "pred": "certificate (paths.check_pred_tree): every pred hop is an input edge on a shortest path, "
                    "no cycles"}


def bench_tiers(lib, nat, h, dist, pred, work, stream, n, args, block, steps=2):
    """The same n=16384 solve on the wider value tiers (the headline runs on the narrowest tier
    the certificate allows, u8 for this graph): forced w32 and i32 on the same int32 input, and
    the continuous-weight fp32 variant (BASELINE C2's variant at this n: the same edge mask with
    U[1, 100) fp32 weights, exact fp32 tier). Each: ms per solve (CUDA events, 1 warm-up) and
    the fraction of its own tier's measured instruction ceiling."""
    import torch

    import paper_2310_03983_b200 as ap

    out = {}
    info = nat.ApspInfo()
    sp = ctypes.c_void_p(stream.cuda_stream)
    hf = None
    for name in ("w32", "i32", "f32_continuous"):
        if name == "f32_continuous":
            hf = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, args.rho, 100, 7 + n))).to(h.device)
            src, dt, tier_req = hf, nat.DTYPE_F32, nat.TIER_AUTO
            dbuf = dist.view(torch.float32)
        else:
            src, dt, tier_req = h, nat.DTYPE_I32, {"w32": nat.TIER_W32, "i32": nat.TIER_I32}[name]
            dbuf = dist
        need = lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, dt, n, block)
        if need > work.numel():
            out[name] = {"skipped": f"workspace {need} B > {work.numel()} B"}
            continue

        def one():
            with torch.cuda.stream(stream):
                dbuf.copy_(src)
            nat.check(lib.apsp_fw_blocked(dt, n, dbuf.data_ptr(), n, pred.data_ptr(), n, block, tier_req,
                                          work.data_ptr(), work.numel(), sp, ctypes.byref(info)))
        one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            one()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        tier = nat.TIER_NAMES[info.tier]
        rate = n ** 3 / (ms / 1e3)
        out[name] = {"tier": tier, "ms_per_step": ms, "value": rate, "unit": UNIT, "steps": steps,
                     "frac_of_tier_ceiling": rate / TIER_PEAK[tier], "tier_ceiling": TIER_PEAK[tier],
                     "op": TIER_OP[tier], "pct_fp32_core_peak": rate / FP32_CORE_PEAK}
        if name == "f32_continuous":
            ok, why = ap.check_pred_paths(hf, dbuf, pred, 1e-5)
            out[name]["pred_paths_resummed_within_1e-5"] = ok
            out[name]["input"] = "generator mask of GenParams(16384, 0.1, 100, 16391), fp32 weights U[1,100) " \
                                 "(paper_2310_03983_b200.continuous_costs)"
    del hf
    return out


def bench_python_api(h_np, n, reps=3):
    """The reference-facing Python call a user of the reference makes: fw_classic on an int64
    CostMatrix (pageable numpy in, frozen int64 ApspSolution out), wall clock per call."""
    import paper_2310_03983_b200 as ap

    h64 = h_np.astype(np.int64)
    h64[h_np == ap.INF32] = ap.INF_RAW   # (np.where with the int32 array would wrap INF_RAW to 0)
    h = ap.CostMatrix(h64, _validated=True)
    ap.fw_classic(h)   # warm-up: staging buffers, pool growth
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        sol = ap.fw_classic(h)
        ts.append(time.perf_counter() - t)
        info = sol.info
        del sol
    dt = statistics.median(ts)
    return {"value": n ** 3 / dt, "unit": UNIT, "ms_per_call": dt * 1e3, "calls": reps,
            "ms_all": [round(x * 1e3, 1) for x in ts], "device_ms": info.get("device_ms"), "tier": info.get("tier"),
            "classic_for_zero_edges": info.get("classic_for_zero_edges"),
            "wire_bytes_per_cell": [info.get("h2d_bytes_per_cell"), info.get("d2h_bytes_per_cell")],
            "api": "paper_2310_03983_b200.fw_classic(CostMatrix) -> ApspSolution (int64, pageable numpy both ways; "
                   "reference solvers.py:118-155 signature)",
            "h2d_bytes_per_call": n * n * 8, "d2h_bytes_per_call": n * n * 16,
            "note": "bytes are those of the int64 host arrays; on the wire they travel narrowed (csrc/hostio.cu)"}


def bench_e2e(lib, nat, h_np, n, args, block):
    """Reference-facing host call: pinned host buffers in/out, copies inside the timed region."""
    import torch

    hin = torch.from_numpy(h_np).pin_memory()
    dout = torch.empty((n, n), dtype=torch.int32).pin_memory()
    pout = torch.empty((n, n), dtype=torch.int32).pin_memory()
    info = nat.ApspInfo()

    def call():
        st = lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, hin.data_ptr(), dout.data_ptr(),
                                 pout.data_ptr(), nat.DTYPE_I32, nat.IDX_PRED, block, 0, 0, nat.TIER_AUTO, 0,
                                 ctypes.byref(info))
        nat.check(st)

    for _ in range(max(1, args.warmup)):
        call()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(args.steps):
        call()
    dt = time.perf_counter() - t
    return {"value": n ** 3 * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": n * n * info.h2d_bytes_per_cell,
            "d2h_bytes_per_step": n * n * info.d2h_bytes_per_cell, "ms_per_step": dt / args.steps * 1e3,
            "api": "apsp_solve_host (C ABI, host buffers; synchronous like the reference solvers)",
            "transfers": "int32 costs in, int32 dist + pred out, in the caller's buffers; both cross PCIe "
                         f"narrowed ({info.h2d_bytes_per_cell} B/cell up, {info.d2h_bytes_per_cell} B/cell down) "
                         "with host threads packing / widening chunks beside the copies (csrc/hostio.cu)"}


if __name__ == "__main__":
    main()
