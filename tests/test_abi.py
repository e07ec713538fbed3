"""CPU tests of the C-ABI library: it loads without a GPU, exports every symbol
include/tarragon.h declares, and its host-side table / mask / version logic
behaves as specified (host-only ctx, device = -1: no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tg():
    import paper_2601_01310_b200 as tg
    return tg


def test_exports_every_declared_symbol():
    tg = _tg()
    hdr = open(os.path.join(ROOT, "include", "tarragon.h")).read()
    declared = set(re.findall(r"\b(tg_[a-z_]+)\s*\(", hdr))
    assert len(declared) >= 15
    lib = ctypes.CDLL(tg.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert declared == set(tg.EXPORTED), declared ^ set(tg.EXPORTED)


def _host_ctx(E=8, W=2, G=1, rank=0, k=2):
    tg = _tg()
    pl = wl.make_placement(E, W, G)
    ctx = tg.tg_init(64, E, k, 128, pl.n_ews, pl.ew_rank, pl.slots_per_ew, 256, rank=rank, world=G, device=-1)
    for ew in range(W):
        for sl, e in enumerate(pl.hosted[ew]):
            if e >= 0:
                tg.tg_load_experts(ctx, ew, sl, e, None, None, None)
    return tg, ctx, pl


def test_invalid_configs():
    tg = _tg()
    with pytest.raises(tg.TarragonError):
        tg.tg_init(60, 8, 2, 128, 1, [0], 8, 16, device=-1)       # d % 64
    with pytest.raises(tg.TarragonError):
        tg.tg_init(64, 8, 9, 128, 1, [0], 8, 16, device=-1)       # k > 8
    with pytest.raises(tg.TarragonError):
        tg.tg_init(64, 8, 2, 128, 2, [0, 3], 8, 16, world=2, device=-1)  # ew on rank 3 of 2
    assert "ew_rank" in tg.tg_last_error(None)


def test_route_table_rules_and_versions():
    """SPEC S:221-225 (versioned ERT), S:334 (candidate must host the expert), S:205 (NoRoute)."""
    tg, ctx, pl = _host_ctx()
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_OK
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_ERR_STALE_VERSION
    assert tg.tg_set_route_table(ctx, 0, pl.cand) == tg.TG_ERR_STALE_VERSION
    bad = pl.cand.copy()
    bad[0, 0] = bad[1, 0]                    # candidate holds another expert
    assert tg.tg_set_route_table(ctx, 2, bad) == tg.TG_ERR_NOT_LOADED
    assert "holds expert" in tg.tg_last_error(ctx)
    assert tg.tg_set_route_table(ctx, 2, wl.flipped(pl.cand)) == tg.TG_OK
    # a table that leaves an expert without an unmasked candidate is rejected
    assert tg.tg_mask_worker(ctx, 1, 1) == tg.TG_OK
    prim_only = np.ascontiguousarray(pl.cand[:, :1, :])
    assert tg.tg_set_route_table(ctx, 3, prim_only) == tg.TG_ERR_NO_ROUTE
    assert tg.tg_set_route_table(ctx, 3, pl.cand) == tg.TG_OK
    tg.tg_finalize(ctx)


def test_mask_semantics_host_only():
    """masking an EW whose experts have shadows keeps every expert routable; masking the
    shadow host too makes the mask call warn NO_ROUTE and the layer call refuse."""
    tg, ctx, pl = _host_ctx(E=8, W=4, G=2)
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_OK
    assert tg.tg_mask_worker(ctx, 2, 1) == tg.TG_OK
    e = int(np.nonzero(pl.cand[:, 0, 0] == 2)[0][0])
    sw = int(pl.cand[e, 1, 0])
    assert tg.tg_mask_worker(ctx, sw, 1) == tg.TG_ERR_NO_ROUTE
    assert tg.tg_moe_layer(ctx, None, None) in (tg.TG_ERR_UNSUPPORTED, tg.TG_ERR_NO_ROUTE)
    assert tg.tg_mask_worker(ctx, sw, 0) == tg.TG_OK  # rejoin
    assert tg.tg_mask_worker(ctx, 2, 0) == tg.TG_OK
    with pytest.raises(tg.TarragonError):
        tg.tg_mask_worker(ctx, 9, 1)
    tg.tg_finalize(ctx)


def test_mask_rank_host_only():
    """NEXT-3a: fail-stopping a rank masks every EW it hosts; experts keep a
    route through shadows on live ranks; a rank cannot mask itself; rejoin is refused (re-provision)."""
    tg, ctx, pl = _host_ctx(E=8, W=2, G=2, rank=0)
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_OK
    with pytest.raises(tg.TarragonError):
        tg.tg_mask_rank(ctx, 0, 1)                      # itself
    with pytest.raises(tg.TarragonError):
        tg.tg_mask_rank(ctx, 2, 1)                      # out of range
    assert tg.tg_mask_rank(ctx, 1, 0) == tg.TG_OK       # unmask of a live rank: no-op
    assert tg.tg_mask_rank(ctx, 1, 1) == tg.TG_OK       # every expert has a shadow on rank 0
    with pytest.raises(tg.TarragonError) as ei:
        tg.tg_mask_rank(ctx, 1, 0)
    assert ei.value.status == tg.TG_ERR_UNSUPPORTED
    with pytest.raises(tg.TarragonError) as ei:
        tg.tg_mask_worker(ctx, 1, 0)                    # EW 1 lives on the failed rank
    assert ei.value.status == tg.TG_ERR_UNSUPPORTED
    # the failed rank's EWs are masked: a table routing only to them is rejected
    prim_only = np.ascontiguousarray(pl.cand[:, :1, :])
    assert tg.tg_set_route_table(ctx, 2, prim_only) == tg.TG_ERR_NO_ROUTE
    tg.tg_finalize(ctx)
    # two EWs per rank, shadows of EW 2's primaries partly on EW 3 (same rank): no route
    tg, ctx, pl = _host_ctx(E=8, W=4, G=2, rank=0)
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_OK
    assert tg.tg_mask_rank(ctx, 1, 1) == tg.TG_ERR_NO_ROUTE
    tg.tg_finalize(ctx)


def test_host_only_ctx_refuses_compute():
    """No CPU fallback: a host-only ctx returns TG_ERR_UNSUPPORTED from tg_moe_layer."""
    tg, ctx, pl = _host_ctx()
    tg.tg_set_route_table(ctx, 1, pl.cand)
    rc = tg._lib.tg_moe_layer(ctx, None, None, 0, None)
    assert rc == tg.TG_ERR_UNSUPPORTED
    assert "no compute path" in tg.tg_last_error(ctx)
    tg.tg_finalize(ctx)


def test_bank_slots_consecutive_per_rank():
    """EWs of one rank get consecutive bank slots in ew order (DESIGN R#11)."""
    tg, ctx, pl = _host_ctx(E=8, W=4, G=2, rank=1)
    S = tg.tg_max_slots(ctx)
    assert S == 2 * pl.slots_per_ew
    assert [tg.tg_bank_slot(ctx, ew, 0) for ew in range(4)] == [0, pl.slots_per_ew, 0, pl.slots_per_ew]
    assert tg.tg_bank_slot(ctx, 0, pl.slots_per_ew) == -1
    tg.tg_finalize(ctx)


def test_kv_store_host_only_refused():
    """NEXT-4: the checkpoint store needs a device (copy engines); host-only ctx refuses it."""
    tg, ctx, pl = _host_ctx()
    with pytest.raises(tg.TarragonError) as ei:
        tg.tg_kv_store_init(ctx, 1 << 20)
    assert ei.value.status == tg.TG_ERR_UNSUPPORTED
    assert tg.tg_kv_committed(ctx) == 0
    tg.tg_finalize(ctx)


def test_failover_and_host_path_host_only():
    """NEXT-1 host-side validation: failure-timeout range; a host-only ctx has no failover, host path
    or fault injection target (no device)."""
    tg, ctx, pl = _host_ctx(E=8, W=2, G=2, rank=0)
    with pytest.raises(tg.TarragonError):
        tg.tg_set_failure_timeout(ctx, 0.0)
    with pytest.raises(tg.TarragonError):
        tg.tg_set_failure_timeout(ctx, 5000.0)
    assert tg.tg_set_failure_timeout(ctx, 50.0) == tg.TG_OK
    assert tg._lib.tg_failover(ctx, None, None, 0, None, None) == tg.TG_ERR_UNSUPPORTED
    assert tg._lib.tg_host_sync(ctx, None) == tg.TG_ERR_UNSUPPORTED
    assert tg.tg_inject_failure(ctx) == tg.TG_OK  # a flag for the next call (none can run here)
    tg.tg_finalize(ctx)


def test_load_experts_guards_active_table_slots():
    """a slot the active route table names for expert e cannot be overwritten with
    another expert (it would silently serve e's tokens with wrong weights); same expert is fine."""
    tg, ctx, pl = _host_ctx()
    assert tg.tg_set_route_table(ctx, 1, pl.cand) == tg.TG_OK
    e0 = pl.hosted[0][0]
    tg.tg_load_experts(ctx, 0, 0, e0, None, None, None)  # reload of the same expert: allowed
    with pytest.raises(tg.TarragonError) as ei:
        tg.tg_load_experts(ctx, 0, 0, (e0 + 1) % 8, None, None, None)
    assert ei.value.status == tg.TG_ERR_INVALID and "route table" in str(ei.value)
    tg.tg_finalize(ctx)


def test_virtual_rank_and_stage_calls_host_only():
    """Host-only ctxs refuse the device-side bootstrap / export entry points."""
    tg, ctx, pl = _host_ctx()
    for fn, args in ((tg.tg_set_stage_export, (1,)), (tg.tg_connect_local, ([ctx],))):
        with pytest.raises(tg.TarragonError) as ei:
            fn(ctx, *args)
        assert ei.value.status == tg.TG_ERR_UNSUPPORTED
    with pytest.raises(tg.TarragonError):
        tg.tg_get_stage(ctx, tg.TG_STAGE_Y)
    # fused virtual-rank launches need device ctxs of ranks 0..world-1 on one device
    assert tg.tg_moe_layer_multi([ctx], [None], [None]) == tg.TG_ERR_INVALID
    tg.tg_finalize(ctx)


def test_peer_handle_carries_layout_signature():
    """The peer handle is the IPC handle plus the layout signature checked at connect time."""
    tg = _tg()
    assert tg.tg_peer_handle_size() >= 64 + 64
