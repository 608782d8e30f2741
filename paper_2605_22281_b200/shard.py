"""Host-side sharding logic for the multi-GPU path.

Rank g owns a contiguous, nnz-balanced block of A rows (the m-partition) and a
contiguous slice of the n-vectors (the n-partition).  The transpose side is
either COLSHARD (T = the transpose of the local A block, formed locally, its
product reduce-scattered) or ROWSHARD (rank g stores rows of the given B on its
n-slice, w all-gathered).  This module only slices host arrays and drives the
ranks; every arithmetic step runs in libsflsqr.so.
"""
from __future__ import annotations

import threading

import numpy as np


def balanced_row_blocks(rowptr: np.ndarray, world: int) -> list:
    """Contiguous row ranges [r0, r1) per rank, balancing nonzeros (ties -> rows)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    nrows = rowptr.size - 1
    nnz = int(rowptr[-1] - rowptr[0])
    bounds = [0]
    for g in range(1, world):
        target = rowptr[0] + (nnz * g) // world if nnz else 0
        r = int(np.searchsorted(rowptr, target, side="left")) if nnz else (nrows * g) // world
        r = min(max(r, bounds[-1]), nrows)
        bounds.append(r)
    bounds.append(nrows)
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


def even_blocks(n: int, world: int) -> list:
    """The library's n-partition for COLSHARD: n0_g = g * ceil(n / world)."""
    per = -(-n // world)
    return [(min(n, g * per), min(n, (g + 1) * per)) for g in range(world)]


def csr_block(rowptr, col, val, r0, r1):
    """(local rowptr rebased to 0, col, val) of rows [r0, r1) (views into col/val)."""
    s, e = int(rowptr[r0]), int(rowptr[r1])
    return np.ascontiguousarray(rowptr[r0:r1 + 1] - s), col[s:e], val[s:e]


def shard_plan(prob, world: int) -> dict:
    """Partition of a gen.Problem over `world` ranks: A rows, T mode and n-slices."""
    a_blocks = balanced_row_blocks(prob.A.rowptr, world)
    if prob.t_mode == "given":
        t_blocks = balanced_row_blocks(prob.T.rowptr, world)
        return dict(a_blocks=a_blocks, t_mode="rowshard", n_blocks=t_blocks)
    return dict(a_blocks=a_blocks, t_mode="colshard", n_blocks=even_blocks(prob.n, world))


def rank_solve(prob, spec, plan, r, world, mx, eta=None, history=1, device=0, knobs=0, **comm):
    """One rank of a sharded solve: its A rows (and T rows when B is given), its slice of b, the whole
    iteration, then (x slice, true_res, sketch_res, info, done, status, gathered x).  `comm` selects the
    transport (local_group= / nccl_id= / ipc_name=)."""
    from .sflsqr import SFLSQR

    s = SFLSQR(method=spec.method, window=spec.window, maxit=mx, orth_mode=spec.orth_mode, tol=spec.tol,
               eta=spec.eta if eta is None else eta, delta_e=prob.delta_e, history=history, device=device,
               use_graph=False, rank=r, world=world, knobs=knobs, **comm)
    a0, a1 = plan["a_blocks"][r]
    arp, acol, aval = csr_block(prob.A.rowptr, prob.A.col, prob.A.val, a0, a1)
    if plan["t_mode"] == "rowshard":
        t0, t1 = plan["n_blocks"][r]
        trp, tcol, tval = csr_block(prob.T.rowptr, prob.T.col, prob.T.val, t0, t1)
        s.set_operator_shard(prob.m, prob.n, a0, a1, arp, acol, aval, t=(trp, tcol, tval), t_rows=(t0, t1))
    else:
        s.set_operator_shard(prob.m, prob.n, a0, a1, arp, acol, aval)
    s.set_sketch(prob.sketch_seed, spec.d, spec.s_nz)
    s.set_precond(spec.precond, spec.p, spec.eps_rel)
    s.set_rhs(np.ascontiguousarray(prob.b[a0:a1]))
    done, status = s.iterate(mx)
    tr, sk = s.get_residual_norms()
    x = s.get_x()
    xg = s.get_x(gathered=True)
    info = s.get_info()
    s.close()
    return (x, tr, sk, info, done, status, xg)


def run_local_group(prob, spec, world: int, maxit=None, device=0, eta=None, history=1, knobs=0):
    """Run one sharded solve with `world` ranks as host threads of this process
    (SFLSQR_COMM_LOCAL) on one device.  Returns (x, true_res, sketch_res, infos)
    with x assembled from the ranks' n-slices."""
    from .sflsqr import LocalGroup

    plan = shard_plan(prob, world)
    grp = LocalGroup(world, device)
    out = [None] * world
    err = [None] * world
    mx = maxit or spec.maxit

    def rank_main(r):
        try:
            out[r] = rank_solve(prob, spec, plan, r, world, mx, eta=eta, history=history, device=device, knobs=knobs,
                                local_group=grp)
        except Exception as exc:  # surfaced to the caller below
            err[r] = exc

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    x = np.zeros(prob.n)
    for r in range(world):
        info = out[r][3]
        x[info["n0"]:info["n0"] + info["n_loc"]] = out[r][0]
    return x, out[0][1], out[0][2], [o[3] for o in out], [(o[4], o[5]) for o in out], out


def run_ipc_processes(config, gen_kwargs, method, world: int, maxit, device=0, eta=0.0, knobs=0, timeout=600):
    """Run one sharded solve with `world` ranks as separate PROCESSES on one device
    (SFLSQR_COMM_IPC: POSIX shared-memory rendezvous, CUDA-IPC peer memory).  Each process
    regenerates the seeded problem (gen.make_problem(config, **gen_kwargs)) and runs
    `python -m paper_2605_22281_b200.shard <args>`; returns the same tuple as run_local_group."""
    import json
    import os
    import subprocess
    import sys
    import tempfile
    import uuid

    name = "/sflsqr_%d_%s" % (os.getpid(), uuid.uuid4().hex[:12])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as tmp:
        procs = []
        for r in range(world):
            arg = dict(config=config, gen_kwargs=gen_kwargs, method=method, world=world, rank=r, maxit=maxit,
                       device=device, eta=eta, knobs=knobs, name=name, out=os.path.join(tmp, "rank%d.npz" % r))
            procs.append(subprocess.Popen([sys.executable, "-m", "paper_2605_22281_b200.shard", json.dumps(arg)],
                                          cwd=root, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
        logs = []
        for p in procs:
            try:
                o, _ = p.communicate(timeout=timeout)
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                raise RuntimeError("a rank process did not finish within %d s" % timeout)
            logs.append(o.decode(errors="replace"))
        for r, p in enumerate(procs):
            if p.returncode != 0:
                raise RuntimeError("rank %d exited %d:\n%s" % (r, p.returncode, logs[r][-4000:]))
        out = []
        for r in range(world):
            with np.load(os.path.join(tmp, "rank%d.npz" % r), allow_pickle=False) as f:
                info = json.loads(str(f["info"]))
                out.append((f["x"], f["tr"], f["sk"], info, bool(f["done"]), int(f["status"]), f["xg"]))
    n = out[0][3]["n"]
    x = np.zeros(n)
    for o in out:
        x[o[3]["n0"]:o[3]["n0"] + o[3]["n_loc"]] = o[0]
    return x, out[0][1], out[0][2], [o[3] for o in out], [(o[4], o[5]) for o in out], out


def run_local_group_subprocess(config, gen_kwargs, method, world: int, maxit, device=0, eta=0.0, knobs=0, timeout=600):
    """run_local_group in a fresh interpreter that regenerates the seeded problem the way the rank
    processes of run_ipc_processes do (same environment, same host libraries): (x, true_res, sketch_res)."""
    import json
    import os
    import subprocess
    import sys
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as tmp:
        arg = dict(mode="local_group", config=config, gen_kwargs=gen_kwargs, method=method, world=world, maxit=maxit,
                   device=device, eta=eta, knobs=knobs, out=os.path.join(tmp, "local.npz"))
        r = subprocess.run([sys.executable, "-m", "paper_2605_22281_b200.shard", json.dumps(arg)], cwd=root,
                           capture_output=True, text=True, timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError("local group process exited %d:\n%s" % (r.returncode, (r.stdout + r.stderr)[-4000:]))
        with np.load(arg["out"]) as f:
            return f["x"], f["tr"], f["sk"]


def _ipc_rank_main(argv):
    import json
    from gen import make_problem

    a = json.loads(argv[0])
    prob = make_problem(a["config"], **a["gen_kwargs"])
    spec = [s for s in prob.solvers if s.method == a["method"]][0]
    if a.get("mode") == "local_group":
        # the in-process rank group from an interpreter set up exactly like the rank processes
        x, tr, sk, _, _, _ = run_local_group(prob, spec, a["world"], maxit=a["maxit"], device=a["device"],
                                             eta=a["eta"], knobs=a["knobs"])
        np.savez(a["out"], x=x, tr=tr, sk=sk)
        return
    plan = shard_plan(prob, a["world"])
    x, tr, sk, info, done, status, xg = rank_solve(prob, spec, plan, a["rank"], a["world"], a["maxit"], eta=a["eta"],
                                                   device=a["device"], knobs=a["knobs"], ipc_name=a["name"])
    info = {k: (v if isinstance(v, (int, float, str, bool)) else np.asarray(v).tolist()) for k, v in info.items()}
    np.savez(a["out"], x=x, tr=tr, sk=sk, xg=xg, done=done, status=status, info=json.dumps(info))


if __name__ == "__main__":
    import sys
    _ipc_rank_main(sys.argv[1:])
