"""World-size-2 gloo tests of the multi-rank host logic (CPU): every rank builds
the same placement, host-only ctxs agree on bank slots and on table / mask
decisions (SPMD), and the oracle's G-rank layout is G-independent per token."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as wl


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_01310_b200 as tg
        import oracle
        pl = wl.make_placement(8, 4, world)
        ctx = tg.tg_init(64, 8, 2, 128, pl.n_ews, pl.ew_rank, pl.slots_per_ew, 64, rank=rank, world=world,
                         device=-1)
        for ew in range(pl.n_ews):
            for sl, e in enumerate(pl.hosted[ew]):
                if e >= 0:
                    tg.tg_load_experts(ctx, ew, sl, e, None, None, None)
        res = [tg.tg_set_route_table(ctx, 1, pl.cand), tg.tg_mask_worker(ctx, 1, 1),
               tg.tg_set_route_table(ctx, 2, wl.flipped(pl.cand)), tg.tg_mask_worker(ctx, 2, 1),
               tg.tg_set_route_table(ctx, 2, pl.cand)]
        banks = [tg.tg_bank_slot(ctx, ew, s) for ew in range(pl.n_ews) for s in range(pl.slots_per_ew)]
        mine = torch.tensor(res + banks + [tg.tg_max_slots(ctx)], dtype=torch.int64)
        allv = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
        same = all(torch.equal(allv[0], v) for v in allv)
        # oracle layout at G ranks: rank r's tokens keep their global positions (G-independent layout)
        sh = wl.CONFIGS["tiny"]
        L = wl.make_layer(sh, 7)
        x = wl.make_tokens(sh, 7)
        args = ([wl.as_u16(a) for a in L.w1], [wl.as_u16(a) for a in L.w3], [wl.as_u16(a) for a in L.w2])
        r2 = oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), sh.k, *args, pl.cand, pl.ew_rank, pl.slots_per_ew,
                          np.zeros(4, np.uint8), G=world)
        pl1 = wl.make_placement(8, 4, 1)
        r1 = oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), sh.k, *args, pl1.cand, pl1.ew_rank, pl1.slots_per_ew,
                          np.zeros(4, np.uint8), G=1)
        same_out = np.array_equal(r1["out"], r2["out"])
        # rows per EW are the same whichever rank hosts it
        rows_g = sum(int(r2["counts"].sum()) for _ in [0])
        t = torch.tensor([float(np.max(np.abs(r2["w"].sum(1) - 1)))])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)          # max over ranks (as bench.py reduces timings)
        q.put((rank, same, res, same_out, rows_g == sh.T * sh.k, float(t.item())))
        tg.tg_finalize(ctx)
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, 29611, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, res, same_out, rows_ok, wmax in out:
        assert same, "ranks disagree on SPMD table/mask decisions or bank slots"
        assert res == [0, 0, 0, -2, -4]           # OK, OK, OK, NO_ROUTE (EW2 holds a shadow of an EW1 expert), STALE
        assert same_out and rows_ok and wmax <= 1e-6
