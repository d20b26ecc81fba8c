#!/usr/bin/env python
"""bench.py — DDELM-NN solve throughput on B200 (driver contract).

A step is one complete DDELM-NN solve of the named BASELINE config (default C3: 8x8
subdomains, M=800, the config BASELINE.json's metric is quoted on at 1/2/4/8 GPUs): feature /
collocation build, batched QR + COD of every K_i and Kbar_i, coarse + Neumann layers, reduced
RHS, the interface CG to rel 1e-9 and the coefficient reconstruction.

  value  subdomains/s with inputs (the seeded feature layers) resident in HBM; device time from
         CUDA events on the library's stream, K steps bracketed by barrier + synchronize.
  e2e    the same through the public C-ABI from the host: reseed (host RNG -> pinned -> H2D),
         solve, D2H of coefficients and mu, every step.

--impl reference times the reference's CPU algorithm (the oracle restatement; the reference
itself cannot be built here) on the host cores, bounded sample + extrapolation.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)



def load_traffic(family):
    """DRAM bytes per launch of `family` from the committed ncu capture (profiles/traffic.json,
    written by tools/summarize_profiles.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(family)
        return {"bytes": t["dram_bytes_per_launch"], "source": t["source"]} if t else None
    except Exception:  # noqa: BLE001
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = 6554.2
    try:
        with open(p) as f:
            hbm = float(json.load(f).get("hbm_gbs", hbm))
    except Exception:  # noqa: BLE001
        pass
    return hbm


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def one_gpu_harness_test() -> bool:
    """DDELM_BENCH_ONE_GPU=1: harness self-test of the N-rank path on ONE GPU (every rank on
    device 0, gloo process group, host-staged exchange). Its timings are not valid numbers — the
    ranks share a GPU — and the JSON line says so (`harness_test`)."""
    return os.environ.get("DDELM_BENCH_ONE_GPU") == "1"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if one_gpu_harness_test() else int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_init(world):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    backend = "nccl" if torch.cuda.is_available() and not one_gpu_harness_test() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend)
    return dist


def _coll_device(dist) -> str:
    import torch
    return "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# --------------------------------------------------------------------------- CPU (oracle)
def cpu_solve(cfg_name: str, cg_workers: int = 1):
    """ONE complete solve of the reference's CPU algorithm on the host (the oracle restatement;
    the reference itself cannot be built here): Workspace build with LsFactor on
    SciPy's LAPACK (dgeqrf / dgeqp3 / dtzrzf, oracle/lapack.cpp; one BLAS thread per call),
    workers = nproc for the per-subdomain setup phases (the reference's only parallel knob,
    solvers.cpp:138,150,286,401), and the interface CG single-threaded as in the reference
    (solvers.cpp:95-117). No extrapolation: the whole solve is timed."""
    from oracle import pyoracle as o
    from paper_2503_10032_b200.configs import CONFIGS

    c = CONFIGS[cfg_name]
    nproc = os.cpu_count() or 1
    lib = o.use_lapack(True)
    try:
        t0 = time.perf_counter()
        ws = o.OracleWorkspace(problem=c["problem"], s=c["s"], n_grid=c["n_grid"], M=c["M"], l=c["l"],
                               seed=c["seed"], flux_variant=c["flux_variant"], trace_basis=c["trace_basis"],
                               workers=nproc, cg_workers=cg_workers)
        t1 = time.perf_counter()
        r = ws.solve(c["method"], c["theta"], c["cg_rel_tol"])
        t2 = time.perf_counter()
    finally:
        o.use_lapack(False)
    tim = {k: round(v, 4) for k, v in r.timings.items()}
    return {"seconds": t2 - t0, "build_s": t1 - t0, "solve_s": t2 - t1, "iterations": int(r.iterations),
            "timings": tim, "cores": nproc, "cg_threads": cg_workers,
            "blas": f"LAPACK from SciPy's OpenBLAS ({os.path.basename(lib)}), 1 thread per call",
            "sample": (f"{cfg_name}: one complete DDELM-NN solve ({2 * c['s'] ** 2} local LS factorisations on "
                       f"{nproc} worker threads, coarse + Neumann layers, {int(r.iterations)} CG iterations "
                       f"on {cg_workers} thread(s) as in the reference, reconstruction); no extrapolation")}


def run_reference(args, cfg, world, rank):
    """The reference arm: complete CPU solves of the workload on the host cores. A solve of C3
    takes tens of seconds on one CG thread, so the run does min(K, budget / first-solve) complete
    solves (at least one) and reports that count as `steps` (steps_requested = K)."""
    if rank != 0:
        return
    nsub = cfg["s"] ** 2
    # warm-up: one complete solve of the smallest config (pages in the oracle and LAPACK)
    cpu_solve("C1")
    secs, last = [], None
    t_start = time.perf_counter()
    while len(secs) < args.steps:
        last = cpu_solve(args.config)
        secs.append(last["seconds"])
        spent = time.perf_counter() - t_start
        if spent + secs[-1] > args.ref_budget_s:
            break
    mean_s = sum(secs) / len(secs)
    value = nsub / mean_s
    line = {"impl": "reference", "metric": "ddelm_nn_solve_throughput", "value": value,
            "unit": "subdomains/s", "n_gpus": args.gpus, "steps": len(secs), "steps_requested": args.steps,
            "warmup": 1, "warmup_note": "one complete C1 solve (a C3 solve is tens of seconds of CPU)",
            "ms_per_step": mean_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args, cfg, 1),
                           parallelism=f"reference CPU path on {last['cores']} host cores (rank 0 of {world})"),
            "cpu_baseline": {"value": value, "unit": "subdomains/s", "cores": last["cores"], "kind": "port",
                             "sample": last["sample"], "blas": last["blas"],
                             "threads": {"setup": last["cores"], "cg": last["cg_threads"]}},
            "e2e": {"value": value, "unit": "subdomains/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "solve_seconds": mean_s, "solve_seconds_each": secs, "detail": last}
    print(json.dumps(line), flush=True)


def lsq_microbench(P, nblocks, device, peak, reps=3):
    """BASELINE config C5: nblocks fp64 blocks [K (3000 x 1000) | B (3000 x 200)] of tanh features,
    batched Householder QR (B carried as appended columns: Q^T B) + Schur block S = B^T B -
    (Q^T B)^T (Q^T B) on DMMA. Device-resident inputs (generated on the GPU), CUDA-event timed."""
    m, n, k = 3000, 1000, 200
    L = P.LsqBatch(nblocks, m, n, k, device)
    L.generate(1, "tanh")
    L.factor()  # warm-up
    qr = sc = 0.0
    for _ in range(reps):
        L.generate(1, "tanh")
        a, b = L.factor()
        qr += a
        sc += b
    qr, sc = qr / reps, sc / reps
    fl = L.flops_per_block() * nblocks
    t = (qr + sc) / 1e3
    tf = fl / t / 1e12
    del L
    return {"config": f"C5: {nblocks} blocks, K {m}x{n} + B {m}x{k}, tanh(w.x+b), fp64",
            "blocks_per_s": nblocks / t, "ms_per_step": qr + sc, "qr_ms": qr, "schur_ms": sc,
            "tflops": tf, "peak_tflops": peak, "frac_fp64_peak": tf / peak,
            "flops_per_block": fl / nblocks,
            "flop_model": "geqrf 2mn^2-2n^3/3 + Q^T B 4mnk-2n^2k + S 2(m-n)k^2 (SURVEY.md §8d)"}


def fact_schur_flops(cfg, ranks, ranks_bar):
    """SURVEY.md §8d algorithmic FP64 work of the local factorisation + Schur / coarse assembly
    (standard LAPACK counts, per-subdomain ranks from the run):
      per local matrix (K_i and Kbar_i): geqrf(m, M) = 2 m M^2 - 2/3 M^3, plus
        COD(m, M, r) = 4 m M r - 2 (m + M) r^2 + 4/3 r^3 + 4 r^2 (M - r)   (deficient branch) or
        orgqr(m, M) = 2 m M^2 - 2/3 M^3                                     (full-rank branch);
      Schur: Ypi / Gpi 2 m M c_i + 2 m r_i c_i (c_i corner columns), Dpp / Dpd 2 m M per
      cross-flux row and owner, S_Pi 2 n_pf n_pi^2."""
    s, M, ng = cfg["s"], cfg["M"], cfg["n_grid"]
    m = ng * ng  # every local grid point is one K (and Kbar) row
    f_fact = 0.0
    for r in list(ranks) + list(ranks_bar):
        f_fact += 2.0 * m * M * M - 2.0 / 3.0 * M ** 3
        if r < M:
            f_fact += 4.0 * m * M * r - 2.0 * (m + M) * r * r + 4.0 / 3.0 * r ** 3 + 4.0 * r * r * (M - r)
        else:
            f_fact += 2.0 * m * M * M - 2.0 / 3.0 * M ** 3
    f_schur = 0.0
    for i, r in enumerate(ranks):
        ix, iy = i % s, i // s
        c = sum(1 for a in (0, 1) for b in (0, 1) if 1 <= ix + a <= s - 1 and 1 <= iy + b <= s - 1)
        f_schur += 2.0 * m * M * c + 2.0 * m * r * c
    n_pi = (s - 1) ** 2
    npf = 2 * n_pi
    f_schur += npf * 2 * (2.0 * m * M) + 2.0 * npf * n_pi ** 2
    return f_fact, f_schur


def fp64_fraction(cfg, ranks, ranks_bar, phase_ms, peak):
    f_fact, f_schur = fact_schur_flops(cfg, ranks, ranks_bar)
    t = (phase_ms["qr"] + phase_ms["cod"] + phase_ms["coarse"]) / 1e3
    tf = (f_fact + f_schur) / t / 1e12
    return {"flops_fact": f_fact, "flops_schur": f_schur, "seconds_fact_schur": t, "tflops": tf,
            "peak_tflops": peak, "frac": tf / peak,
            "formula": "SURVEY.md §8d: (F_fact + F_schur) / t_(qr + cod + coarse phases), LAPACK flop counts"}


def run_single_config(P, name, steps, warmup, stream_of, peak):
    """A second single-GPU bench line (BASELINE config C4: 16x16 subdomains, M = 1000): device-
    resident solves timed with CUDA events, both CG representations."""
    import torch
    c = P.CONFIGS[name]
    ws = P.workspace_from_config(name)
    stream = stream_of(ws)
    cg = P.CgOptions(rel_tol=c["cg_rel_tol"])
    out = {"config": name, "subdomains": c["s"] ** 2, "M": c["M"], "n_grid": c["n_grid"], "l": c["l"],
           "problem": c["problem"]}
    for mode in ("coeff", "compact"):
        ws.set_cg_blocks(mode)
        for _ in range(warmup):
            ws.invalidate()
            ws._solve("ddelm-nn", c["theta"], cg, fetch=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        its = []
        for _ in range(steps):
            ws.invalidate()
            rep = ws._solve("ddelm-nn", c["theta"], cg, fetch=False)
            its.append(rep.iterations)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rk, rkb, _ = ws.ranks()
        d = {"value": c["s"] ** 2 / (ms / 1e3), "unit": "subdomains/s", "ms_per_step": ms, "iterations": its,
             "phase_ms": {k: round(v, 3) for k, v in rep.phase_ms.items()}}
        if mode == "coeff":
            d["fp64_fact_schur"] = fp64_fraction(c, rk, rkb, rep.phase_ms, peak)
            out.update(d)
        else:
            out["cg_compact"] = d
    ws.set_cg_blocks("coeff")
    del ws
    return out


def workload_config(args, cfg, world=1, exchange="nccl"):
    return {"workload": f"{args.config}: DDELM-NN (theta {cfg['theta']}) {cfg['s']}x{cfg['s']} subdomains, "
                        f"M={cfg['M']}, n_grid={cfg['n_grid']}, l={cfg['l']}, {cfg['problem']}, "
                        f"{cfg['flux_variant']} + {cfg['trace_basis']}, cg_rel_tol {cfg['cg_rel_tol']}",
            "subdomains": cfg["s"] ** 2, "neurons_per_subdomain": cfg["M"],
            "collocation_points_per_subdomain": cfg["n_grid"] ** 2,
            "l2_policy": "working set (2N local matrices, >1 GB at C3) far exceeds the 126 MB L2",
            "parallelism": ((f"sharded x{world}: contiguous strip of subdomains per GPU (one process per GPU), "
                             "owner-slot segments over NCCL send/recv between the CG phases, CG loop as "
                             "chunked CUDA graphs") if world > 1 and exchange == "nccl" else
                            (f"sharded x{world}: contiguous strip of subdomains per GPU, owner-slot segments "
                             f"through the {exchange} exchange, host-loop CG driver") if world > 1 else "single GPU")}


# --------------------------------------------------------------------------- ours
def run_ours(args, cfg, world, rank, local, dist):
    import torch

    import paper_2503_10032_b200 as P

    torch.cuda.set_device(local)
    # the FP64 roofline denominator, measured live on this GPU (DMMA loop; ddelm_gpu_fp64_peak)
    fp64_peak = P.fp64_peak(local)
    exchange = "none"
    if world > 1:
        # sharded: this rank owns a strip of subdomains; the owner-slot entries other ranks read
        # move over NCCL send/recv. If NCCL cannot be set up on any rank, every rank falls back —
        # loudly, and labelled in the JSON line — to the host-staged exchange (POSIX shared memory)
        # so the scaling run still completes (DDELM_BENCH_EXCHANGE=host forces it).
        import torch as _t
        ws, err = None, ""
        if os.environ.get("DDELM_BENCH_EXCHANGE", "nccl") != "host" and not one_gpu_harness_test():
            try:
                obj = [P.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                ws = P.workspace_from_config(args.config, device=local, shard=(rank, world, obj[0]))
            except Exception as e:  # noqa: BLE001
                err = f"{type(e).__name__}: {e}"
                print(f"bench.py rank {rank}: NCCL sharded workspace failed ({err})", file=sys.stderr, flush=True)
        bad = _t.tensor([0 if ws is not None else 1], dtype=_t.int32, device=_coll_device(dist))
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()):
            ws = None
            name = f"/ddelm_bench_{os.environ.get('MASTER_PORT', '0')}"
            ws = P.workspace_from_config(args.config, device=local, shard=(rank, world, "host:" + name))
            exchange = "host-staged (NCCL unavailable" + (f": {err[:120]}" if err else " or forced") + ")"
            print(f"bench.py rank {rank}: using the host-staged exchange", file=sys.stderr, flush=True)
        else:
            exchange = "nccl"
    else:
        ws = P.workspace_from_config(args.config, device=local)
    cg = P.CgOptions(rel_tol=cfg["cg_rel_tol"])
    theta = cfg["theta"] if cfg["method"] == "ddelm-nn" else 0.0
    nsub = cfg["s"] ** 2
    M = cfg["M"]
    seed = cfg["seed"]
    stream = torch.cuda.ExternalStream(ws.stream_handle)

    def solve(fetch=True):
        return ws._solve("ddelm-nn" if theta > 0 else "ddelm-cs", theta, cg, fetch=fetch)

    for _ in range(args.warmup):
        ws.reseed(seed)
        solve()
    torch.cuda.synchronize()

    # ---- device-resident throughput (value)
    clocks = ClockSampler(local)
    clocks.start()
    barrier(dist)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters, launches = [], 0
    spans = []
    for _ in range(args.steps):
        ws.invalidate()
        rep = solve(fetch=False)
        iters.append(rep.iterations)
        launches += rep.launches
        spans.append(ws.device_span_ms())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    dev_ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    dev_ms_max = max_over_ranks(dist, dev_ms)
    value = nsub * args.steps / (dev_ms_max / 1e3)  # the whole problem, sharded over the ranks

    # ---- end-to-end through the public API (host buffers, H2D + D2H inside)
    barrier(dist)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        ws.reseed(seed)
        rep = solve()  # includes reading coefficients, mu and the residual history back
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    e2e_ms = max_over_ranks(dist, t0.elapsed_time(t1))
    e2e_value = nsub * args.steps / (e2e_ms / 1e3)
    n_mu = ws.n_delta + ws.n_pi
    h2d = 3 * nsub * M * 8  # seeded feature layers of every subdomain (summed over the ranks)
    d2h = (nsub * M + world * (n_mu + max(rep.iterations, 1))) * 8

    # ---- roofline: one profiled solve with per-kernel-family CUDA events
    ws.set_profiling(True)
    ws.invalidate()
    solve()
    ws.set_profiling(False)
    fam = {}
    for f in ("build_features", "qr_factor", "qr_panel", "qr_trailing", "cod_pivqr", "cod_finish", "cg_iterations"):
        try:
            fam[f] = ws.kernel_stats(f)
        except Exception:  # noqa: BLE001
            pass
    dominant = max(fam.items(), key=lambda kv: kv[1]["ms"])[0] if fam else None
    hbm = load_peaks()
    roof = None
    if dominant:
        s = fam[dominant]
        if s["flops"] > 0:
            ach = s["flops"] / (s["ms"] / 1e3) / 1e12
            tr = load_traffic(dominant)
            roof = {"kernel": dominant, "bound": "tensor", "achieved": ach, "peak": fp64_peak,
                    "unit": "TFLOP/s", "frac": ach / fp64_peak,
                    "peak_source": "FP64 DMMA loop measured live in this run (MEASURED_PEAKS.json carries no "
                                   "FP64 entry)",
                    "traffic": tr["bytes"] if tr else None, "traffic_source": tr["source"] if tr else None,
                    "launches": s["launches"], "avg_launch_ms": s["ms"] / s["launches"]}
        else:
            ach = s["bytes"] / (s["ms"] / 1e3) / 1e9 if s["bytes"] > 0 else None
            tr = load_traffic(dominant)
            roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": (ach / hbm) if ach else None,
                    "traffic": tr["bytes"] if tr else None,
                    "traffic_source": tr["source"] if tr else None,
                    "algorithmic_bytes_per_launch": s["bytes"] / s["launches"],
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs", "launches": s["launches"],
                    "avg_launch_ms": s["ms"] / s["launches"]}
    qr = fam.get("qr_factor") or fam.get("qr_trailing")
    families = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                    "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                    "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
                for k, v in fam.items()}

    # ---- the same solve with the compact interface-level CG blocks (ddelm_gpu_set_cg_blocks):
    # same operator in exact arithmetic, another CG round-off trajectory
    compact = None
    if not args.no_compact:
        ws.set_cg_blocks("compact")
        for _ in range(2):
            ws.invalidate()
            solve(fetch=False)
        barrier(dist)
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        citers = []
        for _ in range(args.steps):
            ws.invalidate()
            crep = solve(fetch=False)
            citers.append(crep.iterations)
        c1.record(stream)
        torch.cuda.synchronize()
        barrier(dist)
        cms = max_over_ranks(dist, c0.elapsed_time(c1)) / args.steps
        t0.record(stream)
        for _ in range(args.steps):
            ws.reseed(seed)
            crep = solve()
        t1.record(stream)
        torch.cuda.synchronize()
        barrier(dist)
        cms_e2e = max_over_ranks(dist, t0.elapsed_time(t1)) / args.steps
        ws.set_profiling(True)
        ws.invalidate()
        solve()
        ws.set_profiling(False)
        cfam = {}
        for f in ("qr_factor", "cod_pivqr", "cod_finish", "cg_iterations"):
            try:
                v = ws.kernel_stats(f)
            except Exception:  # noqa: BLE001
                continue
            if f in fam:  # the stats accumulate over profiled solves: this solve's share only
                v = {k: v[k] - fam[f][k] for k in ("ms", "launches", "flops", "bytes")}
            cfam[f] = {"ms": round(v["ms"], 3),
                       "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                       "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
        compact = {"value": nsub / (cms / 1e3), "unit": "subdomains/s", "ms_per_step": cms,
                   "iterations": citers, "e2e": {"value": nsub / (cms_e2e / 1e3), "unit": "subdomains/s",
                                                 "ms_per_step": cms_e2e},
                   "phase_ms": {k: round(v, 3) for k, v in crep.phase_ms.items()},
                   "kernel_families": cfam,
                   "note": "CG on precomputed interface-level blocks (F [C Ypi])^T, (Cdelta Cbar)^T; "
                           "not the headline: its CG round-off trajectory differs from the reference's"}
        ws.set_cg_blocks("coeff")

    ws_driver, ws_exchange = ws.cg_driver, exchange
    # FP64 roofline of the factorisation + Schur phase by SURVEY.md §8d's formula (the headline
    # solve's own ranks and phase times)
    fp64_frac = None
    if world == 1:
        rk, rkb, _ = ws.ranks()
        fp64_frac = fp64_fraction(cfg, rk, rkb, rep.phase_ms, fp64_peak)
    c4 = None
    if world == 1 and not args.no_c4 and args.config != "C4":
        del ws
        c4 = run_single_config(P, "C4", max(2, min(args.steps, 5)), 2,
                               lambda w: torch.cuda.ExternalStream(w.stream_handle), fp64_peak)
    lsq = None
    if not args.no_lsq and world == 1:
        lsq = lsq_microbench(P, args.lsq_blocks, local, fp64_peak)
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        c = cpu_solve(args.config)
        cpu = {"value": nsub / c["seconds"], "unit": "subdomains/s", "cores": c["cores"], "kind": "port",
               "sample": c["sample"], "blas": c["blas"], "threads": {"setup": c["cores"], "cg": c["cg_threads"]},
               "seconds": c["seconds"], "iterations": c["iterations"], "timings": c["timings"]}
    ms_step = dev_ms_max / args.steps
    line = {"metric": "ddelm_nn_solve_throughput", "value": value, "unit": "subdomains/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded feature layers; manufactured Poisson data)",
            "config": workload_config(args, cfg, world, exchange),
            "solve_seconds": ms_step / 1e3, "iterations": iters,
            "e2e": {"value": e2e_value, "unit": "subdomains/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps},
            "roofline": roof, "kernel_families": families,
            "phase_ms": {k: round(v, 3) for k, v in rep.phase_ms.items()},
            "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk,
            "fp64_lsq_microbench": lsq, "cg_compact": compact, "fp64_fact_schur": fp64_frac,
            "fp64_peak": {"tflops": fp64_peak, "source": "measured live in this run: DMMA m8n8k4 loop on every SM "
                          "(ddelm_gpu_fp64_peak; r01 probe: 37.2, profiles/r01_fp64_peaks.json)"},
            "c4": c4, "cg_driver": ws_driver, "exchange": ws_exchange,
            "fp64_qr_tflops": (qr["flops"] / (qr["ms"] / 1e3) / 1e12) if qr else None}
    if one_gpu_harness_test():
        line["harness_test"] = "DDELM_BENCH_ONE_GPU=1: all ranks shared ONE GPU; timings are not valid numbers"
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: start the N ranks ourselves (one process per GPU,
    torch.distributed.run on 127.0.0.1) and pass their output through."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not one_gpu_harness_test():
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}",
              file=sys.stderr, flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: stop starting new complete CPU solves after this many seconds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compact", action="store_true", help="skip the compact-CG-blocks solve")
    ap.add_argument("--no-lsq", action="store_true", help="skip the C5 local-solve microbenchmark")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (16x16, M=1000) second line")
    ap.add_argument("--lsq-blocks", type=int, default=1024)
    args = ap.parse_args()
    from paper_2503_10032_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return
    dist = dist_init(world)
    run_ours(args, cfg, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
