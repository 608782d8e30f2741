#!/usr/bin/env python3
"""Benchmark of the sketched flexible Golub-Kahan step (BASELINE.json metric).

One "step" = one sFLSQR iteration (all SURVEY.md §8(a) rows a1-a9) of the
config-4 workload (BASELINE.json configs[3]: 1024^2 Siddon CT, 720 angles x
1449 bins, unmatched pixel-driven backprojector B, ell = 4, d = 400, s = 8,
identity tau; the largest configuration that fits one B200 and the one the
metric's 1/2/4/8-GPU scaling is quoted on).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Timing: W untimed warm-up iterations, then
exactly K iterations bracketed by barrier + cuda.synchronize, CUDA events on
the library's stream (torch's current stream), max over ranks.  The operators
(~30 GB) exceed L2 (126 MB), so no L2 flush is needed between iterations.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sFLSQR iterations/s at 1/2/4/8 B200; achieved HBM GB/s vs 8 TB/s/GPU"
UNIT = "iterations/s"
CONTRACT_PEAK_GBS = 8000.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.proc = None
        self.idx = device_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        if not getattr(self, "lines", None):
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


_DIST_DEV = "cuda"   # "cpu" under --comm ipc (gloo process group)


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=_DIST_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


FMT_NAMES = ["CSR", "pair-CSR", "aligned pair-CSR", "interpolation pair-CSR", "sliced-ELL interpolation pairs"]


def _traffic(workload, kernel):
    p = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        d = json.load(open(p))
        return d.get(kernel)
    except Exception:
        return None


def _spec_for(prob, method):
    """The config's solver spec; method "flsqr" / "flsmr" runs the unsketched full-orthogonalisation
    parent with the config's operator, tau and maxit."""
    import dataclasses
    if method is None:
        return prob.solvers[0]
    for x in prob.solvers:
        if x.method == method:
            return x
    if method in ("sflsqr", "sflsmr", "flsqr", "flsmr", "lsqr", "lsmr"):
        return dataclasses.replace(prob.solvers[0], method=method)
    raise SystemExit(f"unknown method {method}")


def _host_cpu():
    """CPU model and usable core count of the host the line was measured on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


def run_cpu_baseline(prob, spec, budget_s=40.0, min_its=5):
    """The oracle as it stands (single thread), first iterations of the same workload: at least
    min_its iterations beyond the first (more when they fit the budget)."""
    from threadpoolctl import threadpool_limits
    from oracle.operators import operator_from_problem
    from oracle.sflsqr import solve_problem
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        op = operator_from_problem(prob)
        t_op = time.perf_counter() - t0
        # one iteration to size the sample, then k iterations inside the budget
        t0 = time.perf_counter()
        solve_problem(prob, spec, op=op, maxit=1, record=False)
        t1 = time.perf_counter() - t0
        k = int(max(min_its + 1, min(spec.maxit, budget_s // max(t1, 1e-6))))
        t0 = time.perf_counter()
        solve_problem(prob, spec, op=op, maxit=k, record=False)
        tk = time.perf_counter() - t0
    per_it = max((tk - t1) / max(k - 1, 1), 1e-9) if k > 1 else t1
    return {"value": 1.0 / per_it, "unit": UNIT, "cores": 1, "kind": "oracle", "host": _host_cpu(),
            "iterations": k - 1,
            "sample": (f"oracle (NumPy + plain C CSR, 1 thread) on the full {prob.name} problem: solve with "
                       f"maxit={k} minus maxit=1, i.e. iterations 2..{k} ({k - 1} iterations; init + first "
                       f"iteration separated); {per_it:.3g} s/iteration, init+1st iteration {t1:.3g} s, "
                       f"operator setup {t_op:.3g} s")}


def bench_reference(args, prob, spec, world, rank):
    """--impl reference: the oracle (this tier's reference arm), bounded sample."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    from oracle.operators import operator_from_problem
    from oracle.sflsqr import solve_problem
    budget = float(os.environ.get("SFLSQR_REF_BUDGET_S", "120"))
    # W warm-up iterations (init + iterations 1..W, untimed beyond sizing), then K iterations timed
    # as the difference of two solves (maxit = W + K minus maxit = W), K capped by the time budget
    W = max(1, args.warmup)
    with threadpool_limits(limits=1):
        op = operator_from_problem(prob)
        t0 = time.perf_counter()
        solve_problem(prob, spec, op=op, maxit=W, record=False)
        tw = time.perf_counter() - t0
        k = int(max(1, min(args.steps, spec.maxit - W, budget // max(tw / (W + 1), 1e-3))))
        t0 = time.perf_counter()
        solve_problem(prob, spec, op=op, maxit=W + k, record=False)
        tk = time.perf_counter() - t0
    per_it = max((tk - tw) / k, 1e-12)
    val = 1.0 / per_it
    line = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": k,
            "warmup": W, "ms_per_step": per_it * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": prob.name, "m": prob.m, "n": prob.n,
                       "nnz_A": prob.A.nnz if prob.A is not None else None,
                       "nnz_T": prob.T.nnz if prob.T is not None else (prob.A.nnz if prob.A is not None else None),
                       "ell": spec.window, "d": spec.d,
                       "s": spec.s_nz, "tau": spec.precond},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "host": _host_cpu(),
                             "sample": (f"{k} oracle iterations ({W + 1}..{W + k}) of the full workload after init + "
                                        f"{W} warm-up iterations (time budget {budget:.0f} s for the timed part)")},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=195)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default=None,
                    help="sflsqr | sflsmr | flsqr | flsmr | lsqr | lsmr (default: the config's first; flsqr/flsmr = unsketched, "
                         "full orthogonalisation)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="graph replay without per-kernel events")
    ap.add_argument("--N", type=int, default=None, help="override grid size (debug)")
    ap.add_argument("--no-windows", action="store_true", help="skip the late-window and full-solve timings")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1 transport: nccl (one GPU per rank, the measured configuration) or ipc (process ranks "
                         "over CUDA-IPC peer memory with a host rendezvous, ranks mapped round-robin onto the visible "
                         "devices: runs the sharded branch on fewer GPUs than ranks, a functional check, not a "
                         "scaling number)")
    ap.add_argument("--knobs", default="", help="comma-separated opts.knobs names (A/B runs; default: none)")
    args = ap.parse_args()

    world, rank, local = _dist()
    from gen import make_problem
    from gen.problems import CONFIGS
    if args.impl == "reference":
        if rank != 0:
            return            # the reference arm runs on rank 0 only
        prob = make_problem(args.config, **(dict(N=args.N) if args.N else {}))
        spec = _spec_for(prob, args.method)
        bench_reference(args, prob, spec, world, rank)
        return

    import torch
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        sys.exit(1)
    if args.comm == "ipc":
        global _DIST_DEV
        _DIST_DEV = "cpu"
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    # a dedicated non-default stream: the library issues on it and the CUDA events below record on it
    torch.cuda.set_stream(torch.cuda.Stream())
    if world > 1:
        import torch.distributed as dist
        if args.comm == "ipc":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_22281_b200 import solver_for_problem
    from paper_2605_22281_b200._build import build_library
    if rank == 0:
        build_library()
    _barrier(world)

    W, K = args.warmup, args.steps
    knobs = [k for k in args.knobs.split(",") if k]
    sharded = world > 1 and CONFIGS[args.config]["kind"] == "ct" and not args.N
    t_gen = time.perf_counter()
    if sharded:
        # every rank generates and holds only its A (and B) row block
        from gen.problems import ct_row_nnz, make_ct_shard
        from paper_2605_22281_b200.shard import balanced_row_blocks
        from paper_2605_22281_b200.sflsqr import SFLSQR, get_unique_id
        import torch.distributed as dist

        def allreduce_sum(v):
            t = torch.tensor([v], dtype=torch.float64, device=_DIST_DEV)
            dist.all_reduce(t)
            return float(t.item())

        a_cnt, t_cnt = ct_row_nnz(args.config)
        ab = balanced_row_blocks(np.concatenate([[0], np.cumsum(a_cnt)]), world)
        tb = None if t_cnt is None else balanced_row_blocks(np.concatenate([[0], np.cumsum(t_cnt)]), world)
        prob = make_ct_shard(args.config, ab[rank], None if tb is None else tb[rank], allreduce_sum)
        spec = _spec_for(prob, args.method)
        t_gen = time.perf_counter() - t_gen
        uid = torch.zeros(128, dtype=torch.uint8, device=_DIST_DEV)
        if rank == 0:
            if args.comm == "ipc":   # the group's POSIX shm name, NUL padded
                raw = ("/sflsqr_bench_%d_%d" % (os.getpid(), time.time_ns() % 10**9)).encode().ljust(128, b"\0")
            else:
                raw = get_unique_id()
            uid.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm_kw = (dict(ipc_name=bytes(uid.cpu().numpy()).rstrip(b"\0").decode()) if args.comm == "ipc"
                   else dict(nccl_id=bytes(uid.cpu().numpy())))
        maxit = max(spec.maxit, W + K)
        t_up = time.perf_counter()
        s = SFLSQR(method=spec.method, window=spec.window, maxit=maxit, orth_mode=spec.orth_mode, tol=spec.tol,
                   eta=0.0, delta_e=prob.delta_e, device=local, use_graph=True, rank=rank, world=world,
                   knobs=knobs, **comm_kw)
        A = prob.A_loc
        t = None if prob.T_loc is None else (prob.T_loc.rowptr, prob.T_loc.col, prob.T_loc.val)
        s.set_operator_shard(prob.m, prob.n, prob.a_rows[0], prob.a_rows[1], A.rowptr, A.col, A.val, t=t,
                             t_rows=prob.t_rows or (0, 0))
        s.set_sketch(prob.sketch_seed, spec.d, spec.s_nz)
        s.set_precond(spec.precond, spec.p, spec.eps_rel)
        t_up = time.perf_counter() - t_up
        b_host = prob.b_loc
        nnz_A = int(allreduce_sum(float(A.nnz)))
        nnz_T = int(allreduce_sum(float(prob.T_loc.nnz if prob.T_loc is not None else A.nnz)))
        transport = "NCCL" if args.comm == "nccl" else \
            f"CUDA-IPC process ranks on {min(world, torch.cuda.device_count())} device(s), host rendezvous"
        parallelism = f"shard{world} ({'ROWSHARD' if prob.T_loc is not None else 'COLSHARD'}, {transport})"
    else:
        prob = make_problem(args.config, **(dict(N=args.N) if args.N else {}))
        spec = _spec_for(prob, args.method)
        t_gen = time.perf_counter() - t_gen
        maxit = max(spec.maxit, W + K)
        t_up = time.perf_counter()
        s = solver_for_problem(prob, spec, maxit=maxit, eta=0.0, device=local, use_graph=True, knobs=knobs)
        t_up = time.perf_counter() - t_up
        b_host = prob.b
        nnz_A = prob.A.nnz if prob.A is not None else None
        nnz_T = prob.T.nnz if prob.T is not None else nnz_A
        parallelism = "replicas" if world > 1 else "single"
    stream = torch.cuda.current_stream()

    def timed_region(profiled, W=W, K=K):
        """W untimed iterations, then exactly K timed ones between barrier + synchronize."""
        s.set_rhs(b_host)                              # (re)start the solve
        s.iterate(W)                                   # untimed warm-up
        b_w = s.get_info()["bytes_model"]              # SURVEY.md §8(d) bytes of iteration W
        s.set_profiling(profiled)
        s.reset_profile()
        l0 = s.get_info()["launches"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _barrier(world)
        torch.cuda.synchronize()
        with ClockSampler(local) as ck:
            e0.record(stream)
            dn, stt = s.iterate(K)
            e1.record(stream)
            torch.cuda.synchronize()
        _barrier(world)
        t_ms = _max_over_ranks(e0.elapsed_time(e1), world)
        pr = s.get_profile()
        s.set_profiling(False)
        inf = s.get_info()
        if inf["k_done"] != W + K:
            # a stop inside the window would leave launches that return early: refuse the number
            raise SystemExit(f"bench: the solve stopped at k = {inf['k_done']} inside the timed window "
                             f"{W + 1}..{W + K} (status {inf['status']})")
        # §8(d) bytes are affine in k: the sum over k = W+1..W+K from iterations W and W+K
        b_k = inf["bytes_model"]
        s8d = K * (b_w + (b_k - b_w) / K + b_k) / 2.0 if W >= 1 else K * b_k
        return dict(ms=t_ms, launches=inf["launches"] - l0, prof=pr, clk=ck, done=dn, status=stt, s8d_bytes=s8d,
                    rank_flag=inf["rank_flag"])

    # (1) production timing: one CUDA graph per iteration (single rank) / eager with NCCL (sharded)
    R1 = timed_region(False)
    ms, launches, clk, done, status = R1["ms"], R1["launches"], R1["clk"], R1["done"], R1["status"]
    # (2) the same K iterations again with CUDA events around every launch (per-kernel times)
    R2 = timed_region(True) if not args.no_profile else None
    ms_prof, prof, clk2 = (R2["ms"], R2["prof"], R2["clk"]) if R2 else (None, {}, None)
    # (3) costs that grow with k (x reconstruction, W-path residual): the last 20 iterations of the
    #     maxit solve, and the whole solve averaged (iterations 1..maxit), same launch mode as (1)
    windows = {}
    if not args.no_windows and maxit > 20:
        RL = timed_region(False, W=maxit - 20, K=20)
        RF = timed_region(False, W=1, K=maxit - 1)
        for nm, R, lo, hi in (("late", RL, maxit - 19, maxit), ("full_solve", RF, 2, maxit)):
            kk = hi - lo + 1
            windows[nm] = {"iterations": f"{lo}..{hi}", "value": (kk if sharded else kk * world) / (R["ms"] / 1e3),
                           "ms_per_step": R["ms"] / kk, "step_gbs_s8d": R["s8d_bytes"] / (R["ms"] / 1e3) / 1e9,
                           "clocks": R["clk"].summary()}
    info_end = s.get_info()
    k_done = info_end["k_done"]
    # sharded: the ranks cooperate on one solve (iterations/s of the job); replicas: independent solves
    value = (K if sharded else K * world) / (ms / 1e3)

    # roofline of the dominant kernel (HBM-bound SpMV), on two byte bases:
    #   s8d:    SURVEY.md §8(d)'s per-unit figure, 12 B per stored nonzero of the CSR operator + int64 row
    #           pointers + one read of the gathered vector + one write of the product (the contract's basis)
    #   format: the bytes of the storage format the product actually runs on (pair formats are smaller)
    peak, peak_src = _peaks()
    roof = None
    kernels = {}
    inf = s.get_info()
    for nm, d in prof.items():
        if d["launches"]:
            kernels[nm] = {"ms_total": d["ms"], "launches": d["launches"],
                           "ms_per_launch": d["ms"] / d["launches"],
                           "algo_gbs": d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else None,
                           "share": d["ms"] / ms_prof}
    s8d_per_launch = {}
    if inf["nnz_a"]:
        s8d_per_launch["spmv_A"] = 12.0 * inf["nnz_a"] + 8.0 * (inf["m_loc"] + 1) + 8.0 * inf["n"] + 8.0 * inf["m_loc"]
        s8d_per_launch["spmv_T"] = 12.0 * inf["nnz_t"] + 8.0 * (inf["n_loc"] + 1) + 8.0 * inf["m"] + 8.0 * inf["n_loc"]
    if kernels:
        dom = max(kernels, key=lambda k2: kernels[k2]["ms_total"])
        d = prof[dom]
        t_launch = d["ms"] / d["launches"] / 1e3
        bpl = d["bytes"] / d["launches"]
        ach_fmt = bpl / t_launch / 1e9
        b8 = s8d_per_launch.get(dom, bpl)
        ach = b8 / t_launch / 1e9
        fnames = dict(enumerate(FMT_NAMES))
        fmt = {"spmv_A": fnames[inf["a_fmt"]], "spmv_T": fnames[inf["t_fmt"]]}
        tkey = dom + {"CSR": "", "pair-CSR": "_pcsr", "aligned pair-CSR": "_apcsr",
                      "interpolation pair-CSR": "_ipcsr", "sliced-ELL interpolation pairs": "_sell"}[fmt.get(dom, "CSR")]
        tr = _traffic(prob.name, tkey)
        l1 = _traffic(prob.name, tkey + "_l1_wavefronts_pct")
        kname = {"spmv_A": f"k_spmv_csr_pf, {fmt['spmv_A']} (A z)",
                 "spmv_T": f"k_spmv_csr_pf, {fmt['spmv_T']} (T w)"}.get(dom, dom)
        roof = {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "bytes_basis": "SURVEY.md §8(d): 12 B per stored nonzero (int32 col + fp64 value) of the CSR "
                               "operator + 8 B int64 row pointers + one read of the gathered vector + one write "
                               "of the product",
                "algorithmic_bytes_per_launch": b8,
                "format_bytes_per_launch": bpl, "achieved_format_bytes": ach_fmt, "frac_format_bytes": ach_fmt / peak,
                "format_bytes_basis": f"bytes of the format the product runs on ({fmt.get(dom, 'CSR')}): CSR 12 B/nnz, "
                                      "pair-CSR 20 B per adjacent-column pair (interpolation pairs 12 B) + 12 B per "
                                      "singleton, + row pointers and vectors (DESIGN.md §5)",
                "peak_source": peak_src, "launch_ms": t_launch * 1e3, "traffic": tr,
                "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch (profiles/)",
                "l1_wavefronts_pct_of_peak": l1,
                "note": ("this product's gathers keep the L1 data pipe at l1_wavefronts_pct_of_peak (ncu), so inside "
                         "the power-capped loop it follows the SM clock" if (l1 or 0) > 70 else "HBM bound")}
    fmt_step_bytes = sum(d["bytes"] for d in prof.values())
    # step throughput on both bases, over the production-timed region (1)
    step = {"s8d_gbs": R1["s8d_bytes"] / (ms / 1e3) / 1e9,
            "format_gbs": (fmt_step_bytes / (ms / 1e3) / 1e9) if fmt_step_bytes else None}
    step["s8d_frac_of_peak"] = step["s8d_gbs"] / peak
    step["s8d_frac_of_8TBs"] = step["s8d_gbs"] / CONTRACT_PEAK_GBS
    step["format_frac_of_peak"] = step["format_gbs"] / peak if step["format_gbs"] else None
    step["note"] = ("s8d: SURVEY.md §8(d)'s byte model of the whole step (CSR operators at 12 B/nnz, vectors, "
                    "x reconstruction, W-path residual) over the production time; it can exceed the copy peak "
                    "because the products run on lossless smaller formats (format: the bytes those formats and "
                    "the other kernels actually move, from the per-kernel model of DESIGN.md §5)")

    # e2e through the public API: host b -> set_rhs, K iterations, x + histories back to host
    e2e = None
    if not args.no_e2e:
        b_pin = torch.from_numpy(np.ascontiguousarray(b_host)).pin_memory()
        x_pin = torch.empty(s.n, dtype=torch.float64).pin_memory()
        _barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.set_rhs(b_pin)
        s.iterate(K)
        s.get_x(x_pin)
        tr_hist, sk_hist = s.get_residual_norms()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        te = _max_over_ranks(te, world)
        e2e = {"value": (K if sharded else K * world) / te, "unit": UNIT,
               "h2d_bytes_per_step": 8.0 * len(b_host) / K, "d2h_bytes_per_step": (8.0 * s.n + 16.0 * K) / K,
               "note": "set_rhs(pinned host b) + iterate(K) + get_x(pinned host) + get_residual_norms, wall clock"}
    s.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(prob, spec)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": prob.name, "method": spec.method, "m": prob.m, "n": prob.n,
                       "nnz_A": nnz_A, "nnz_T": nnz_T,
                       "spmv_format": {"A": FMT_NAMES[info_end["a_fmt"]], "T": FMT_NAMES[info_end["t_fmt"]],
                                       "pairs_A": info_end["a_pairs"], "pairs_T": info_end["t_pairs"]},
                       "ell": spec.window, "d": spec.d, "s": spec.s_nz, "tau": spec.precond, "maxit": maxit,
                       "iterations_timed": f"{W + 1}..{W + K}", "history": "true residual (W path) on",
                       "l2": "inputs larger than L2 (operators ~30 GB vs 126 MB L2); no flush",
                       "parallelism": parallelism, "knobs": knobs,
                       **({"functional_check_only": "process ranks share device(s): not a scaling measurement"}
                          if (sharded and args.comm == "ipc" and world > torch.cuda.device_count()) else {}),
                       "launch": ("CUDA graph per iteration" + (" (NCCL collectives captured)" if sharded else ""))
                                 if info_end["graph"] else "eager launches" + ((" + NCCL" if args.comm == "nccl" else
                                                                                " + host-rendezvous collectives") if sharded else ""),
                       "per_kernel_timing": "second timed region of K iterations, eager launches with CUDA events "
                                            "on the library stream (ms_per_step_profiled)"},
            "roofline": roof,
            "step": step,
            "windows": windows,
            "ms_per_step_profiled": (ms_prof / K) if ms_prof else None,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "clocks_profiled_region": clk2.summary() if clk2 else None,
            "kernels": kernels,
            "status": {"done": done, "status": status, "k_done": k_done, "rank_flag": R1["rank_flag"],
                       "rank_flag_note": "1: a projected problem had |R_kk| < 1e-14 max|R_jj| (reading R14); the "
                                         "timed iterations then run on a numerically rank-deficient sketched basis"},
            "host": _host_cpu(),
            "setup_s": {"generate": t_gen, "upload": t_up},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
