"""CPU tests (gloo, world_size 2 and 3) of the sharded DDELM-NN host logic.

The sharded device path (ddelm_gpu_create_sharded) runs one strip of subdomains per GPU and
exchanges every cross-subdomain sum as a SUM all-reduce of owner-slot tables. Correctness rests on
two properties of the host-side plan (plan.cpp shard_plan), checked here across real processes:
  1. every slot of every table has exactly one writer among all ranks, and the union of the
     strips' writers is exactly the single-device writer set (same slot, same subdomain-local
     position);
  2. the all-reduce of per-rank send tables (zeros in non-owned slots) reproduces the
     single-device table bit for bit (x + 0 = x), whatever the reduction order.
The device kernels are the same on one or many GPUs; the GPU test suite checks the phase-by-phase
path with world = 1 against the persistent kernel bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2503_10032_b200 as P

CFGS = ["T2", "C2", "C3", "T3b"]  # T3b: biharmonic, two components per interface point


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tables_as_writers(cfg, rank, world):
    """Global-size int tables: entry = global writer id (sub * width + pos) + 1 at the slots this
    rank writes, 0 elsewhere."""
    t = P.plan_tables(cfg, rank, world)
    out = {}
    sizes = {"gamma_dst": 2 * t["n_delta"], "flux_dst": 2 * t["n_delta"], "nd_dst": 2 * t["n_delta"],
             "corner_dst": 4 * t["n_pi"], "cross_dst": 4 * t["npf"]}
    widths = {"gamma_dst": t["gmax"], "flux_dst": t["fmax"], "nd_dst": t["dmax"], "corner_dst": t["ncq"],
              "cross_dst": t["crmax"]}
    for name, size in sizes.items():
        w = np.zeros(max(size, 1), dtype=np.int64)
        cnt = np.zeros(max(size, 1), dtype=np.int64)
        dst = t[name]
        for k, d in enumerate(dst):
            if d >= 0:
                sub = t["sub_lo"] + k // widths[name]
                w[d] = sub * widths[name] + k % widths[name] + 1
                cnt[d] += 1
        out[name] = (w, cnt)
    return out, t


def _worker(rank, world, port, cfg_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.CONFIGS[cfg_name]
        mine, t = _tables_as_writers(cfg, rank, world)
        ref, _ = _tables_as_writers(cfg, 0, 1)
        ok = {}
        for name, (w, cnt) in mine.items():
            tw, tc = torch.from_numpy(w.copy()), torch.from_numpy(cnt.copy())
            dist.all_reduce(tw)
            dist.all_reduce(tc)
            rw, rc = ref[name]
            # property 1: one writer per used slot, the same writer as on one device
            ok[name] = bool((tc.numpy() == rc).all() and (tc.numpy() <= 1).all() and (tw.numpy() == rw).all())
        # property 2: a synthetic exchange of float tables (values keyed by the writer) is exact
        rng = np.random.default_rng(123)
        vals = rng.standard_normal(2 * t["n_delta"] * 2 + 1)
        w, _ = mine["gamma_dst"]
        send = np.where(w > 0, vals[w % len(vals)], 0.0)
        ts = torch.from_numpy(send)
        dist.all_reduce(ts)
        rw, _ = ref["gamma_dst"]
        expect = np.where(rw > 0, vals[rw % len(vals)], 0.0)
        ok["exchange_exact"] = bool(np.array_equal(ts.numpy(), expect))
        # the strips tile the subdomains
        lo, hi = P.shard_range(t["n_global"], rank, world)
        ok["strip"] = (lo, hi) == (t["sub_lo"], t["sub_lo"] + t["n_local"])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg_name", CFGS)
def test_owner_slots_partition_over_ranks(cfg_name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok in res:
        assert all(ok.values()), (rank, ok)


def test_shard_ranges_cover_all_subdomains():
    for n in (4, 16, 64, 256):
        for world in (1, 2, 3, 4, 8):
            strips = [P.shard_range(n, r, world) for r in range(world)]
            assert strips[0][0] == 0 and strips[-1][1] == n
            assert all(strips[r][1] == strips[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in strips) - min(b - a for a, b in strips) <= 1
