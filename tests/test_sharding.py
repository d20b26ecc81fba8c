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


# ------------------------------------------------------------------ exchange plan (XPlan)
def _touched_delta(t):
    """Delta indices of this rank's subdomains (the readers of a Delta slot table)."""
    return {int(d) // 2 for d in t["gamma_dst"] if d >= 0}


def _writer_slots(t):
    """Global slots this rank writes, per exchange table (plan.hpp XTable)."""
    g = {int(d) for d in t["gamma_dst"] if d >= 0}
    f = {int(d) for d in t["flux_dst"] if d >= 0}
    n = {int(d) for d in t["nd_dst"] if d >= 0}
    c = {int(d) for d in t["corner_dst"] if d >= 0}
    x = {int(d) for d in t["cross_dst"] if d >= 0}
    pap = set(range(t["sub_lo"], t["sub_lo"] + t["n_local"]))
    return {"t": c, "psi": x, "t3": c, "o": g, "x": f, "tr": n, "zz": n, "xc": x, "opi": c, "pap": pap}


def _slot_value(table, slot):
    return float(np.sin(1.0 + 7.0 * P.XTABLES.index(table) + 0.37 * slot))


def _xworker(rank, world, port, cfg_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.CONFIGS[cfg_name]
        t = P.plan_tables(cfg, rank, world)
        mine = _writer_slots(t)
        touched = _touched_delta(t)
        allw = [None] * world
        dist.all_gather_object(allw, mine)
        ok = {}
        for one in (False, True):
            xl = P.exchange_lists(cfg, rank, world, one_level=one)
            every = [None] * world
            dist.all_gather_object(every, xl)
            for name in P.XPOINTS:
                L = xl[name]
                # the segments this rank receives from q are exactly what q sends to it, in order
                for q_ in range(world):
                    if q_ == rank:
                        continue
                    Lq = every[q_][name]
                    so = int(Lq["soff"][rank])
                    sent = Lq["send"][so:so + int(Lq["scnt"][rank])]
                    ro = int(np.sum(L["rcnt"][:q_]))
                    got = L["recv"][ro:ro + int(L["rcnt"][q_])]
                    ok[f"{one}/{name}/pair{q_}"] = bool(np.array_equal(sent, got))
                    # every slot q sends is written by q
                    ok[f"{one}/{name}/writer{q_}"] = all(int(s) in allw[q_][P.XTABLES[int(tb)]] for tb, s in sent)
                # simulated exchange: local writes + imports reproduce the single-device table on
                # every slot this rank reads
                tabs = {}
                for tb, s in L["recv"]:
                    tabs.setdefault(P.XTABLES[int(tb)], {})[int(s)] = _slot_value(P.XTABLES[int(tb)], int(s))
                for tname in {P.XTABLES[int(tb)] for tb, _ in np.concatenate([L["recv"], L["send"]])} if len(L["recv"]) + len(L["send"]) else set():
                    have = dict(tabs.get(tname, {}))
                    for s_ in mine[tname]:
                        have[s_] = _slot_value(tname, s_)
                    written = set().union(*[allw[r][tname] for r in range(world)])
                    if tname in ("x", "tr", "zz"):
                        need = {s_ for s_ in written if s_ // 2 in touched}
                    else:
                        need = written
                    ok[f"{one}/{name}/{tname}/complete"] = need <= set(have)
                    ok[f"{one}/{name}/{tname}/values"] = all(have[s_] == _slot_value(tname, s_) for s_ in need)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg_name", ["T2", "C2", "T3b"])
def test_exchange_plan_over_ranks(cfg_name, world):
    """Pairwise send/receive lists agree, every sent slot is written by its sender, and a rank's
    own writes plus its imports cover every slot it reads (Delta tables: the indices its
    subdomains touch; coarse and O / pap tables: all) — the exchange reproduces the single-device
    tables on every slot a consumer reads."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xworker, args=(r, world, port, cfg_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok in res:
        bad = [k for k, v in ok.items() if not v]
        assert not bad, (rank, bad[:10])


def test_exchange_plan_world1_is_empty():
    xl = P.exchange_lists(P.CONFIGS["T2"], 0, 1)
    assert all(len(xl[n]["send"]) == 0 and len(xl[n]["recv"]) == 0 for n in P.XPOINTS)
