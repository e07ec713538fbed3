"""Multi-GPU parity of tg_moe_layer (run under torchrun, one rank per GPU).

    torchrun --nproc-per-node G --master-addr 127.0.0.1 --master-port P tests/mp_parity.py [--config tiny] [--W W]

Every rank is an AW shard (contiguous token block) and hosts W/G logical EWs
with spread shadows.  Checks: routing and the permutation of the
rank's tokens bit-exact vs the oracle at G ranks, outputs within tolerance,
masked EW (+ NaN poison) and route flips bit-identical, run-to-run bitwise,
and (P7) the G-rank output bitwise equal to a 1-GPU run of the same layer.
Rank 0 prints one JSON line with the report and exits non-zero on failure.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as wl  # noqa: E402
from parity_util import check, collect  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--W", type=int, default=0, help="logical EWs (default = world)")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--sample", type=int, default=0, help="oracle FFN on this many sampled tokens (0 = all)")
    ap.add_argument("--rank-fail", action="store_true",
                    help="fail-stop the last rank (tg_mask_rank) instead of the EW/flip checks")
    ap.add_argument("--empty-rank", action="store_true",
                    help="the last rank calls with 0 tokens: the others' outputs must not change")
    ap.add_argument("--inflight-fail", action="store_true",
                    help="the last rank crashes mid-call; survivors repair that call (tg_failover)")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2601_01310_b200 as tg

    sh = wl.CONFIGS[a.config]
    T = a.tokens or sh.T
    assert T % world == 0
    Tr = T // world
    W = a.W or world
    seed = 3000
    L = wl.make_layer(sh, seed)
    x = wl.make_tokens(sh, seed, T)
    pl = wl.make_placement(sh.E, W, world)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tr, rank=rank, world=world, device=local,
                        group=dist.group.WORLD)
    if os.environ.get("TG_NO_EXPORT") != "1":
        layer.export_stages(True)
    xr = x[rank * Tr:(rank + 1) * Tr].contiguous().to(dev)
    rep = {"rank": rank, "world": world, "W": W, "config": a.config, "T": T}
    ok = True
    msgs = []

    def run():
        o = layer(xr)
        torch.cuda.synchronize()
        return o

    def gather(o):
        outs = [torch.empty_like(o) for _ in range(world)]
        dist.all_gather(outs, o)
        return torch.cat(outs).cpu()

    out = run()
    out_all = gather(out)
    # every rank's routing and stage exports -> rank 0, which checks them all against the oracle
    views = [None] * world
    dist.all_gather_object(views, collect(layer, out, t0=rank * Tr))
    if rank == 0:
        if a.sample:
            rng = np.random.default_rng(seed)
            tok = np.sort(rng.choice(T, size=min(a.sample, T), replace=False)).astype(np.int32)
        else:
            tok = None
        try:
            rep["parity"] = check(views, L, x, pl, [0] * W, tokens=tok, n_threads=min(32, os.cpu_count() or 1))
        except AssertionError as e:
            ok = False
            msgs.append(f"parity: {e}")
    del views
    # determinism.  Rank 0 just spent seconds in the CPU oracle: meet first, else the other
    # ranks' count exchange outlasts its detection timeout (10 x failure timeout, header
    # tg_failover) and they serve this call with rank 0 recorded as failed.
    dist.barrier()
    out2 = run()
    if not torch.equal(out.view(torch.int16), out2.view(torch.int16)):
        ok = False
        dif = out.view(torch.int16) != out2.view(torch.int16)
        toks = dif.any(dim=1).nonzero().flatten()
        same_as_gathered = bool(torch.equal(out2.cpu().view(torch.int16),
                                            out_all[rank * Tr:(rank + 1) * Tr].view(torch.int16)))
        msgs.append(f"rank {rank}: run-to-run differs ({int(dif.sum())} elements, tokens {toks[:6].tolist()} of "
                    f"{int(toks.numel())}; second call equal to the gathered first: {same_as_gathered})")
    if a.rank_fail:
        ok = rank_fail_checks(a, tg, layer, pl, sh, W, rank, world, dev, out, run, msgs, rep) and ok
        finish(ok, rank, rep, msgs, layer, dev)
        return
    if a.empty_rank:
        ok = empty_rank_checks(tg, layer, rank, world, out, xr, dev, msgs, rep) and ok
        finish(ok, rank, rep, msgs, layer, dev)
        return
    if a.inflight_fail:
        ok = inflight_fail_checks(tg, layer, rank, world, out, run, xr, msgs, rep) and ok
        finish(ok, rank, rep, msgs, layer, dev)
        return
    # mask EW1 (+ poison its slots on its rank) -> bit-identical
    ew = 1 % W
    layer.mask_worker(ew, 1)
    if pl.ew_rank[ew] == rank:
        nan = torch.full((sh.F, sh.d), float("nan"), dtype=torch.bfloat16, device=dev)
        nan2 = torch.full((sh.d, sh.F), float("nan"), dtype=torch.bfloat16, device=dev)
        for sl, e in enumerate(pl.hosted[ew]):
            if e >= 0:
                tg.tg_load_experts(layer.ctx, ew, sl, e, nan, nan, nan2)
    else:
        for sl, e in enumerate(pl.hosted[ew]):
            if e >= 0:
                tg.tg_load_experts(layer.ctx, ew, sl, e, None, None, None)
    st0 = layer.stats()
    dist.barrier()
    out_m = run()
    st1 = layer.stats() - st0
    if not torch.equal(out.view(torch.int16), out_m.view(torch.int16)):
        ok = False
        msgs.append(f"rank {rank}: masked output differs ({int((out != out_m).sum())} elements)")
    bank = [tg.tg_bank_slot(layer.ctx, w_, 0) for w_ in range(W)]
    for sl in range(pl.slots_per_ew):
        if st1[pl.ew_rank[ew], bank[ew] + sl] != 0:
            ok = False
            msgs.append(f"rank {rank}: masked EW received rows")
    # rejoin is not possible after poisoning: flip to shadows-first with EW1 still masked
    for i in range(4):
        cand = wl.flipped(pl.cand) if i % 2 == 0 else pl.cand
        layer.set_route_table(cand)
        o = run()
        if not torch.equal(out.view(torch.int16), o.view(torch.int16)):
            ok = False
            msgs.append(f"rank {rank}: flip {i} differs")
    # P7: same layer on one GPU (rank 0), all tokens, W logical EWs
    dist.barrier()
    if rank == 0:
        pl1 = wl.make_placement(sh.E, W, 1)
        one = tg.MoELayer(sh, pl1, L, max_tokens_per_rank=T, rank=0, world=1, device=local)
        o1 = one(x.to(dev))
        torch.cuda.synchronize()
        rep["cross_G_bit_identical"] = bool(torch.equal(o1.cpu().view(torch.int16), out_all.view(torch.int16)))
        one.close()
    finish(ok, rank, rep, msgs, layer, dev)


def rank_fail_checks(a, tg, layer, pl, sh, W, rank, world, dev, out, run, msgs, rep):
    """NEXT-3a (§3.3, §5.2): the last rank fail-stops (stops calling the
    layer; its EWs go with it).  The survivors mask it and keep serving: never waiting on it
    (a wait would trap after the 4 s bounded timeout), never sending it rows, and producing
    outputs for their own tokens bit-identical to the all-alive run (its experts are served by
    their shadows on live ranks, R#8 column independence)."""
    ok = True
    dead = world - 1
    dist.barrier()
    if rank != dead:
        rc = layer.mask_rank(dead)
        if rc != tg.TG_OK:
            return False
        st0 = layer.stats()
        for i in range(6):
            o = run()
            if not torch.equal(out.view(torch.int16), o.view(torch.int16)):
                ok = False
                msgs.append(f"rank {rank}: call {i} after rank {dead} failed differs "
                            f"({int((out != o).sum())} elements)")
        st1 = layer.stats() - st0
        if int(st1[dead].sum()) != 0:
            ok = False
            msgs.append(f"rank {rank}: rows were sent to the failed rank")
        # rejoin is re-provisioning (out of scope): refused
        try:
            layer.mask_rank(dead, 0)
            ok = False
            msgs.append(f"rank {rank}: unmask of a failed rank not refused")
        except tg.TarragonError as e:
            if e.status != tg.TG_ERR_UNSUPPORTED:
                ok = False
                msgs.append(f"rank {rank}: unmask refused with {e}")
        rep["rank_fail_calls"] = 6
    rep["rank_fail_dead"] = dead
    # the failed process is still alive for the harness: it meets the survivors only here
    dist.barrier()
    return ok


def empty_rank_checks(tg, layer, rank, world, out, xr, dev, msgs, rep):
    """A rank with no tokens still takes part in the count exchange and serves its EWs; every
    other rank's outputs are bitwise those of the full call (outputs do not depend on the layout)."""
    ok = True
    empty = world - 1
    for i in range(3):
        if rank == empty:
            e = torch.empty(0, xr.shape[1], dtype=xr.dtype, device=dev)
            rc = tg.tg_moe_layer(layer.ctx, e, torch.empty_like(e))
            torch.cuda.synchronize()
            if rc != tg.TG_OK:
                ok = False
                msgs.append(f"rank {rank}: empty call rc {rc}")
        else:
            o = layer(xr)
            torch.cuda.synchronize()
            if not torch.equal(out.view(torch.int16), o.view(torch.int16)):
                ok = False
                msgs.append(f"rank {rank}: output changed when rank {empty} had no tokens")
    # and back to a full call
    o = layer(xr)
    torch.cuda.synchronize()
    if not torch.equal(out.view(torch.int16), o.view(torch.int16)):
        ok = False
        msgs.append(f"rank {rank}: full call after empty calls differs")
    rep["empty_rank"] = empty
    return ok


def inflight_fail_checks(tg, layer, rank, world, out, run, xr, msgs, rep):
    """NEXT-1 (§5.1): the last rank crashes in the middle of a call (after its count
    exchange and dispatch, before its expert outputs).  Survivors detect it within that call
    (failure timeout on its combine flag), and tg_failover recomputes the pairs they had sent it
    to the next live candidate of each expert on whichever surviving rank hosts it: the repaired
    output of THAT call must be bitwise the unfailed output, at any G (cross-rank replay)."""
    import time
    ok = True
    dead = world - 1
    tg.tg_set_failure_timeout(layer.ctx, 50.0)
    dist.barrier()
    if rank == dead:
        tg.tg_inject_failure(layer.ctx)
        layer(xr)
        torch.cuda.synchronize()
        rep["inflight_dead"] = dead
    else:
        t0 = time.perf_counter()
        o = layer(xr)
        rc, failed = layer.failover(xr, o)
        torch.cuda.synchronize()
        rep["failover_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
        if failed != (1 << dead):
            ok = False
            msgs.append(f"rank {rank}: failed mask {failed:#x}, expected {1 << dead:#x}")
        if rc != tg.TG_OK:
            ok = False
            msgs.append(f"rank {rank}: failover rc {rc}")
        if not torch.equal(out.view(torch.int16), o.view(torch.int16)):
            ok = False
            msgs.append(f"rank {rank}: repaired output differs ({int((out != o).sum())} elements)")
        # the next calls run without the dead rank (fail-stop, NEXT-3a)
        for i in range(3):
            o2 = run()
            if not torch.equal(out.view(torch.int16), o2.view(torch.int16)):
                ok = False
                msgs.append(f"rank {rank}: call {i} after the failover differs")
        rc2, f2 = layer.failover(xr, o2)
        if f2 != 0:
            ok = False
            msgs.append(f"rank {rank}: spurious failure {f2:#x} after masking")
        rep["inflight_rc"] = int(rc)
    dist.barrier()
    return ok


def finish(ok, rank, rep, msgs, layer, dev):
    flags = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flags)
    all_msgs = [None] * dist.get_world_size()
    dist.all_gather_object(all_msgs, msgs)  # every rank's messages, not only rank 0's
    if rank == 0:
        rep["ok"] = bool(flags.item() == 0)
        rep["errors"] = [m for ms in all_msgs for m in ms]
        print(json.dumps(rep), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flags.item() == 0 else 1)


if __name__ == "__main__":
    main()
