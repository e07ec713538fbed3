"""Python binding of libtarragon.so (include/tarragon.h) — argument marshalling only.

Every step of the MoE-layer round trip (gate, ERT resolve, permute, dispatch,
expert FFN, combine) runs in the library's sm_100a kernels.  PyTorch supplies
device memory, streams and (for world > 1) the process group that carries the
peer-handle all-gather.  There is no CPU fallback: if the library is missing
this module raises on import, and a ctx created without a GPU (device = -1)
refuses to compute.

Functions keep the C names (tg_init, tg_load_experts, tg_set_route_table,
tg_mask_worker, tg_moe_layer, ...); ``MoELayer`` bundles them for one layer.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TG_LIB_PATH") or os.path.join(_HERE, "libtarragon.so")  # override: A/B timing only

TG_OK, TG_ERR_INVALID, TG_ERR_NO_ROUTE, TG_ERR_NOT_LOADED = 0, -1, -2, -3
TG_ERR_STALE_VERSION, TG_ERR_CUDA, TG_ERR_PEER, TG_ERR_OOM, TG_ERR_UNSUPPORTED = -4, -5, -6, -7, -8
STATUS = {0: "TG_OK", -1: "TG_ERR_INVALID", -2: "TG_ERR_NO_ROUTE", -3: "TG_ERR_NOT_LOADED",
          -4: "TG_ERR_STALE_VERSION", -5: "TG_ERR_CUDA", -6: "TG_ERR_PEER", -7: "TG_ERR_OOM",
          -8: "TG_ERR_UNSUPPORTED"}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2601_01310_b200/build.py` "
                      "(there is no CPU fallback)")


class tg_config(ctypes.Structure):
    _fields_ = [("d_model", ctypes.c_int), ("n_experts", ctypes.c_int), ("top_k", ctypes.c_int),
                ("d_ffn", ctypes.c_int), ("d_ffn_shared", ctypes.c_int), ("n_ews", ctypes.c_int),
                ("ew_rank", ctypes.POINTER(ctypes.c_int32)), ("slots_per_ew", ctypes.c_int),
                ("max_tokens_per_rank", ctypes.c_int), ("gate_mode", ctypes.c_int), ("shared_gate", ctypes.c_int)]


_lib = ctypes.CDLL(LIB_PATH)
_P, _I, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64
_SIG = {
    "tg_init": ([ctypes.POINTER(tg_config), _I, _I, _I, ctypes.POINTER(_P)], _I),
    "tg_peer_handle_size": ([], ctypes.c_size_t),
    "tg_get_peer_handle": ([_P, _P], _I),
    "tg_connect_peers": ([_P, _P], _I),
    "tg_connect_local": ([_P, _P], _I),
    "tg_moe_layer_multi": ([_P, _I, _P, _P, _P, _P], _I),
    "tg_failover_multi": ([_P, _I, _P, _P, _P, _P, _P], _I),
    "tg_set_stage_export": ([_P, _I], _I),
    "tg_get_stage": ([_P, _I, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)], _I),
    "tg_load_gate": ([_P, _P, _I], _I),
    "tg_load_experts": ([_P, _I, _I, _I, _P, _P, _P, _I], _I),
    "tg_load_shared": ([_P, _P, _P, _P, _I], _I),
    "tg_load_shared_gate": ([_P, _P, _I], _I),
    "tg_set_route_table": ([_P, _U64, _P, _I], _I),
    "tg_mask_worker": ([_P, _I, _I], _I),
    "tg_mask_rank": ([_P, _I, _I], _I),
    "tg_set_failure_timeout": ([_P, ctypes.c_double], _I),
    "tg_failover": ([_P, _P, _P, _I, _P, ctypes.POINTER(ctypes.c_uint32)], _I),
    "tg_inject_failure": ([_P], _I),
    "tg_kv_store_init": ([_P, ctypes.c_size_t], _I),
    "tg_kv_checkpoint": ([_P, _P, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64, _P], _I),
    "tg_kv_committed": ([_P, ctypes.POINTER(ctypes.c_uint64)], _I),
    "tg_kv_restore": ([_P, _P, ctypes.c_size_t, ctypes.c_size_t, _P], _I),
    "tg_moe_layer": ([_P, _P, _P, _I, _P], _I),
    "tg_moe_layer_host": ([_P, _P, _P, _I, _P], _I),
    "tg_host_sync": ([_P, _P], _I),
    "tg_get_routing": ([_P, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "tg_max_slots": ([_P], _I),
    "tg_bank_slot": ([_P, _I, _I], _I),
    "tg_get_stats": ([_P, _P], _I),
    "tg_set_profiling": ([_P, _I], _I),
    "tg_get_kernel_times": ([_P, _P, ctypes.POINTER(_I)], _I),
    "tg_last_launch_count": ([_P], _I),
    "tg_set_trace": ([_P, _I], _I),
    "tg_get_trace": ([_P, _P, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "tg_last_error": ([_P], ctypes.c_char_p),
    "tg_finalize": ([_P], _I),
}
for _n, (_a, _r) in _SIG.items():
    _f = getattr(_lib, _n)
    _f.argtypes, _f.restype = _a, _r

EXPORTED = tuple(_SIG)

TG_STAGE_LOGITS, TG_STAGE_RECV, TG_STAGE_META, TG_STAGE_H, TG_STAGE_Y = 0, 1, 2, 3, 4
TG_STAGE_HSH, TG_STAGE_YSH, TG_STAGE_SGATE = 5, 6, 7


class TarragonError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        assert t.is_contiguous(), "tensors passed to libtarragon must be contiguous"
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    return int(t)


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(ctx, rc: int, what: str, ok=(TG_OK,)):
    if rc not in ok:
        raise TarragonError(rc, f"{what}: {tg_last_error(ctx)}")
    return rc


# ----------------------------------------------------------------- C-name API

def tg_last_error(ctx) -> str:
    return _lib.tg_last_error(ctx).decode()


def tg_init(d_model, n_experts, top_k, d_ffn, n_ews, ew_rank: Sequence[int], slots_per_ew,
            max_tokens_per_rank, rank=0, world=1, device=None, d_ffn_shared=0, gate_mode=0, shared_gate=0):
    """Create a ctx; device=None -> torch.cuda.current_device(); device=-1 -> host-only ctx."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else -1
    ew = (ctypes.c_int32 * len(ew_rank))(*ew_rank)
    cfg = tg_config(d_model, n_experts, top_k, d_ffn, d_ffn_shared, len(ew_rank), ew, slots_per_ew,
                    max_tokens_per_rank, gate_mode, shared_gate)
    h = _P()
    rc = _lib.tg_init(ctypes.byref(cfg), rank, world, device, ctypes.byref(h))
    _check(None, rc, "tg_init")
    return h


def tg_peer_handle_size() -> int:
    return _lib.tg_peer_handle_size()


def tg_get_peer_handle(ctx) -> bytes:
    buf = ctypes.create_string_buffer(tg_peer_handle_size())
    _check(ctx, _lib.tg_get_peer_handle(ctx, buf), "tg_get_peer_handle")
    return buf.raw


def tg_connect_peers(ctx, handles: bytes):
    _check(ctx, _lib.tg_connect_peers(ctx, handles), "tg_connect_peers")


def tg_connect_local(ctx, ctxs):
    """Map the ctxs of every rank (same process, same device) as ctx's peers."""
    arr = (_P * len(ctxs))(*[c.value if isinstance(c, _P) else c for c in ctxs])
    _check(ctx, _lib.tg_connect_local(ctx, arr), "tg_connect_local")


def _ptrs(seq):
    return (_P * len(seq))(*[(c.value if isinstance(c, _P) else c) for c in seq])


def tg_moe_layer_multi(ctxs, xs, outs, stream=None) -> int:
    """One call of every virtual rank of one GPU in one launch; xs[r] None = rank r absent."""
    n = len(ctxs)
    T = (ctypes.c_int * n)(*[(-1 if x is None else x.shape[0]) for x in xs])
    return _lib.tg_moe_layer_multi(_ptrs(ctxs), n, _ptrs([_ptr(x) or 0 for x in xs]),
                                   _ptrs([_ptr(o) or 0 for o in outs]), T, _stream(stream))


def tg_failover_multi(ctxs, xs, outs, stream=None):
    """tg_failover of every virtual rank in one launch: (status, [failed-rank mask per rank])."""
    n = len(ctxs)
    T = (ctypes.c_int * n)(*[(-1 if x is None else x.shape[0]) for x in xs])
    f = (ctypes.c_uint32 * n)()
    rc = _lib.tg_failover_multi(_ptrs(ctxs), n, _ptrs([_ptr(x) or 0 for x in xs]),
                                _ptrs([_ptr(o) or 0 for o in outs]), T, _stream(stream), f)
    return rc, list(f)


def tg_set_stage_export(ctx, on=True):
    _check(ctx, _lib.tg_set_stage_export(ctx, int(on)), "tg_set_stage_export")


_STAGE_DTYPE = {0: np.float32, 1: np.uint16, 2: np.int32, 3: np.uint16, 4: np.uint16, 5: np.uint16, 6: np.uint16,
                7: np.float32}


def tg_get_stage(ctx, stage: int) -> np.ndarray:
    """Flat host copy of a stage value of the last call (see include/tarragon.h)."""
    n = ctypes.c_size_t(0)
    _check(ctx, _lib.tg_get_stage(ctx, stage, None, 0, ctypes.byref(n)), "tg_get_stage")
    dt = np.dtype(_STAGE_DTYPE[stage])
    buf = np.empty(n.value // dt.itemsize, dt)
    if n.value:
        _check(ctx, _lib.tg_get_stage(ctx, stage, buf.ctypes.data, n.value, ctypes.byref(n)), "tg_get_stage")
    return buf


def tg_load_gate(ctx, wg: torch.Tensor):
    _check(ctx, _lib.tg_load_gate(ctx, _ptr(wg), int(wg.is_cuda)), "tg_load_gate")


def tg_load_experts(ctx, ew, slot, expert_id, w1, w3, w2):
    on_dev = int(w1 is not None and isinstance(w1, torch.Tensor) and w1.is_cuda)
    _check(ctx, _lib.tg_load_experts(ctx, ew, slot, expert_id, _ptr(w1), _ptr(w3), _ptr(w2), on_dev),
           "tg_load_experts")


def tg_load_shared(ctx, w1, w3, w2):
    _check(ctx, _lib.tg_load_shared(ctx, _ptr(w1), _ptr(w3), _ptr(w2), int(w1.is_cuda)), "tg_load_shared")


def tg_load_shared_gate(ctx, wsg):
    _check(ctx, _lib.tg_load_shared_gate(ctx, _ptr(wsg), int(wsg.is_cuda)), "tg_load_shared_gate")


def tg_set_route_table(ctx, version: int, cand: np.ndarray) -> int:
    """cand int32 [E, C, 2]; returns the status (raises only on INVALID)."""
    cand = np.ascontiguousarray(cand, dtype=np.int32)
    return _lib.tg_set_route_table(ctx, int(version), cand.ctypes.data, cand.shape[1])


def tg_mask_worker(ctx, ew: int, masked: int = 1) -> int:
    """Returns TG_OK or TG_ERR_NO_ROUTE (warning: mask applied, some expert unroutable)."""
    rc = _lib.tg_mask_worker(ctx, ew, masked)
    return _check(ctx, rc, "tg_mask_worker", ok=(TG_OK, TG_ERR_NO_ROUTE))


def tg_mask_rank(ctx, rank: int, masked: int = 1) -> int:
    """Fail-stop a whole rank (AW + its EWs); returns TG_OK or TG_ERR_NO_ROUTE (warning)."""
    rc = _lib.tg_mask_rank(ctx, rank, masked)
    return _check(ctx, rc, "tg_mask_rank", ok=(TG_OK, TG_ERR_NO_ROUTE))


def tg_set_failure_timeout(ctx, ms: float) -> int:
    return _check(ctx, _lib.tg_set_failure_timeout(ctx, float(ms)), "tg_set_failure_timeout")


def tg_inject_failure(ctx) -> int:
    return _check(ctx, _lib.tg_inject_failure(ctx), "tg_inject_failure")


def tg_failover(ctx, x: torch.Tensor, out: torch.Tensor, stream=None):
    """In-call failover after a tg_moe_layer: returns (status, failed rank mask)."""
    f = ctypes.c_uint32(0)
    rc = _lib.tg_failover(ctx, _ptr(x), _ptr(out), x.shape[0] if x is not None else 0, _stream(stream),
                          ctypes.byref(f))
    _check(ctx, rc, "tg_failover", ok=(TG_OK, TG_ERR_NO_ROUTE))
    return rc, int(f.value)


def tg_kv_store_init(ctx, nbytes: int) -> int:
    return _check(ctx, _lib.tg_kv_store_init(ctx, int(nbytes)), "tg_kv_store_init")


_KV_PENDING = {}  # ctx -> [(seq, tensor)]: segments kept alive until their commit record


def tg_kv_checkpoint(ctx, seg: torch.Tensor, offset: int, seq: int, stream=None) -> int:
    """Checkpoint the device tensor `seg` (contiguous) at bucket offset `offset` with sequence number seq.
    A reference to `seg` is kept until seq is committed (the copy runs later on the checkpoint stream);
    the caller must not modify `seg` before tg_kv_committed() >= seq."""
    nbytes = seg.numel() * seg.element_size()
    rc = _check(ctx, _lib.tg_kv_checkpoint(ctx, _ptr(seg), nbytes, int(offset), int(seq), _stream(stream)),
                "tg_kv_checkpoint")
    key = ctx.value if isinstance(ctx, _P) else ctx
    done = tg_kv_committed(ctx)
    pend = [(q, t) for q, t in _KV_PENDING.get(key, []) if q > done]
    pend.append((int(seq), seg))
    _KV_PENDING[key] = pend
    return rc


def tg_kv_committed(ctx) -> int:
    v = ctypes.c_uint64(0)
    _check(ctx, _lib.tg_kv_committed(ctx, ctypes.byref(v)), "tg_kv_committed")
    return int(v.value)


def tg_kv_restore(ctx, dst: torch.Tensor, offset: int, stream=None) -> int:
    nbytes = dst.numel() * dst.element_size()
    return _check(ctx, _lib.tg_kv_restore(ctx, _ptr(dst), nbytes, int(offset), _stream(stream)), "tg_kv_restore")


def tg_moe_layer(ctx, x: torch.Tensor, out: torch.Tensor, stream=None) -> int:
    n = x.shape[0] if x is not None else 0
    return _lib.tg_moe_layer(ctx, _ptr(x), _ptr(out), n, _stream(stream))


def tg_host_sync(ctx, stream=None) -> int:
    """`stream` waits for every pending host-path copy (outputs of tg_moe_layer_host complete)."""
    return _check(ctx, _lib.tg_host_sync(ctx, _stream(stream)), "tg_host_sync")


def tg_moe_layer_host(ctx, x_host: torch.Tensor, out_host: torch.Tensor, stream=None) -> int:
    return _lib.tg_moe_layer_host(ctx, _ptr(x_host), _ptr(out_host), x_host.shape[0], _stream(stream))


def tg_get_routing(ctx, n_tokens, k, world, S_max, device, stream=None):
    """Routing of the last call (n_tokens must be that call's token count)."""
    idx = torch.empty(n_tokens, k, dtype=torch.int32, device=device)
    w = torch.empty(n_tokens, k, dtype=torch.float32, device=device)
    dr = torch.empty(n_tokens, k, dtype=torch.int32, device=device)
    ds = torch.empty(n_tokens, k, dtype=torch.int32, device=device)
    dp = torch.empty(n_tokens, k, dtype=torch.int32, device=device)
    counts = torch.empty(world, S_max, dtype=torch.int32, device=device)
    _check(ctx, _lib.tg_get_routing(ctx, int(n_tokens), _ptr(idx), _ptr(w), _ptr(dr), _ptr(ds), _ptr(dp),
                                    _ptr(counts), _stream(stream)), "tg_get_routing")
    return dict(idx=idx, w=w, dst_rank=dr, dst_slot=ds, dst_pos=dp, counts=counts)


def tg_max_slots(ctx) -> int:
    return _lib.tg_max_slots(ctx)


def tg_bank_slot(ctx, ew, slot) -> int:
    return _lib.tg_bank_slot(ctx, ew, slot)


def tg_get_stats(ctx, world, S_max) -> np.ndarray:
    rows = np.zeros((world, S_max), np.int64)
    _check(ctx, _lib.tg_get_stats(ctx, rows.ctypes.data), "tg_get_stats")
    return rows


def tg_set_profiling(ctx, on=True):
    _check(ctx, _lib.tg_set_profiling(ctx, int(on)), "tg_set_profiling")


def tg_get_kernel_times(ctx):
    ms = (ctypes.c_float * 8)()
    n = _I(0)
    _check(ctx, _lib.tg_get_kernel_times(ctx, ms, ctypes.byref(n)), "tg_get_kernel_times")
    return [ms[i] for i in range(n.value)]


def tg_set_trace(ctx, on=True):
    _check(ctx, _lib.tg_set_trace(ctx, int(on)), "tg_set_trace")


def tg_get_trace(ctx, cap=1 << 20):
    """Last call's GEMM trace: dict(end ns[n_units], kind[n_units], smid[n_units], start ns[n_ctas],
    front_stamps ns[16]) — end stamps keep the low 48 bits of globaltimer."""
    tr = np.zeros(cap, np.uint64)
    nu, nc = _I(0), _I(0)
    _check(ctx, _lib.tg_get_trace(ctx, tr.ctypes.data, cap, ctypes.byref(nu), ctypes.byref(nc)), "tg_get_trace")
    nu, nc = nu.value, nc.value
    t = tr[:nu]
    m48 = np.uint64((1 << 48) - 1)
    return dict(end=(t >> np.uint64(16)).astype(np.int64),
                kind=((t >> np.uint64(12)) & np.uint64(0xF)).astype(np.int64),
                smid=(t & np.uint64(0xFFF)).astype(np.int64),
                start=(tr[nu:nu + nc] & m48).astype(np.int64),
                front_stamps=(tr[nu + 148:nu + 148 + 64] & m48).astype(np.int64),
                front_stamps_raw=tr[nu + 148:nu + 148 + 64].astype(np.int64),
                front_block_p1=(tr[nu + 148 + 64:nu + 148 + 64 + 148] & m48).astype(np.int64),
                front_block_router=(tr[nu + 148 + 64 + 552:nu + 148 + 64 + 700] & m48).astype(np.int64),
                front_block_prefetch=(tr[nu + 148 + 64 + 700:nu + 148 + 64 + 848] & m48).astype(np.int64),
                topk_detail=tr[nu + 148 + 64 + 1000:nu + 148 + 64 + 1012].astype(np.int64),
                item_clock=tr[nu + 148 + 64 + 1012:nu + 148 + 64 + 1016].astype(np.int64),
                front_block_bar1=(tr[nu + 148 + 64 + 848:nu + 148 + 64 + 996] & m48).astype(np.int64),
                topk_cycles=tr[nu + 148 + 64 + 256:nu + 148 + 64 + 256 + 296].astype(np.int64).reshape(148, 2))


def tg_last_launch_count(ctx) -> int:
    return _lib.tg_last_launch_count(ctx)


def tg_finalize(ctx):
    if ctx:
        _KV_PENDING.pop(ctx.value if isinstance(ctx, _P) else ctx, None)
        _lib.tg_finalize(ctx)


KERNEL_NAMES = ("layer",)


# ----------------------------------------------------------------- convenience

class MoELayer:
    """One MoE layer on this rank: ctx + weights + route table.

    placement: object with n_ews, ew_rank, slots_per_ew, hosted[ew][slot], cand
    (see workloads.make_placement).  weights: object with wg, w1, w3, w2 lists
    (torch bf16, host or device) and optional shared = (w1s, w3s, w2s).
    For world > 1 pass an initialised torch.distributed process group: the
    peer handles are all-gathered through it.  ``local_ranks`` builds the
    ranks of a world as virtual ranks on one GPU instead (see that function).
    """

    def __init__(self, shape, placement, weights, max_tokens_per_rank, rank=0, world=1, device=None,
                 group=None, version=1, _peers=None):
        self.shape, self.pl = shape, placement
        self.rank, self.world = rank, world
        self.stage_export = False
        self.device = torch.cuda.current_device() if device is None else device
        self.ctx = tg_init(shape.d, shape.E, shape.k, shape.F, placement.n_ews, placement.ew_rank,
                           placement.slots_per_ew, max_tokens_per_rank, rank, world, self.device,
                           d_ffn_shared=shape.F_sh, gate_mode=getattr(shape, "gate_mode", 0),
                           shared_gate=getattr(shape, "shared_gate", 0))
        if _peers is not None:
            _peers.append(self.ctx)
            if len(_peers) == world:  # the last virtual rank connects everyone
                for c in _peers:
                    tg_connect_local(c, _peers)
        elif world > 1:
            import torch.distributed as dist
            h = tg_get_peer_handle(self.ctx)
            t = torch.frombuffer(bytearray(h), dtype=torch.uint8).to(f"cuda:{self.device}")
            outs = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(outs, t, group=group)
            blob = b"".join(bytes(o.cpu().numpy().tobytes()) for o in outs)
            tg_connect_peers(self.ctx, blob)
            dist.barrier(group=group)
        tg_load_gate(self.ctx, weights.wg.contiguous())
        for ew in range(placement.n_ews):
            local = placement.ew_rank[ew] == rank
            for sl, e in enumerate(placement.hosted[ew]):
                if e < 0:
                    continue
                if local:
                    tg_load_experts(self.ctx, ew, sl, e, weights.w1[e].contiguous(), weights.w3[e].contiguous(),
                                    weights.w2[e].contiguous())
                else:
                    tg_load_experts(self.ctx, ew, sl, e, None, None, None)
        if shape.F_sh:
            tg_load_shared(self.ctx, *(w.contiguous() for w in weights.shared))
        if getattr(shape, "shared_gate", 0):
            tg_load_shared_gate(self.ctx, weights.wsg.contiguous())
        self.version = 0
        self.set_route_table(placement.cand, version)
        self.S_max = tg_max_slots(self.ctx)

    def set_route_table(self, cand, version=None):
        version = self.version + 1 if version is None else version
        rc = tg_set_route_table(self.ctx, version, cand)
        if rc == TG_OK:
            self.version = version
        return rc

    def mask_worker(self, ew, masked=1):
        return tg_mask_worker(self.ctx, ew, masked)

    def mask_rank(self, rank, masked=1):
        return tg_mask_rank(self.ctx, rank, masked)

    def failover(self, x: torch.Tensor, out: torch.Tensor, stream=None):
        """After a call: repair `out` if an EW failed mid-call; returns (status, failed rank mask)."""
        return tg_failover(self.ctx, x, out, stream)

    def __call__(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(x)
        rc = tg_moe_layer(self.ctx, x, out, stream)
        _check(self.ctx, rc, "tg_moe_layer")
        return out

    def stage(self, which: int) -> np.ndarray:
        return tg_get_stage(self.ctx, which)

    def export_stages(self, on=True):
        """Parity tests: also export the router logits of each call (TG_STAGE_LOGITS)."""
        tg_set_stage_export(self.ctx, on)
        self.stage_export = bool(on)

    def routing(self, n_tokens, stream=None):
        return tg_get_routing(self.ctx, n_tokens, self.shape.k, self.world, self.S_max,
                              f"cuda:{self.device}", stream)

    def stats(self):
        return tg_get_stats(self.ctx, self.world, self.S_max)

    def close(self):
        tg_finalize(self.ctx)
        self.ctx = None

    def __del__(self):
        try:
            if self.ctx:
                self.close()
        except Exception:
            pass


def local_ranks(shape, placement, weights, max_tokens_per_rank, world, device=None):
    """``world`` (<= 4) virtual ranks of one layer on ONE GPU (tests / driver evidence of the
    multi-rank data plane): ctxs connected by device pointer (tg_connect_local); their calls
    run as one cooperative launch (``call_all``: tg_moe_layer_multi)."""
    device = torch.cuda.current_device() if device is None else device
    peers = []
    layers = [None] * world
    # every ctx must exist before any is connected: create, then load (connect happens on the last init)
    for r in range(world):
        layers[r] = MoELayer(shape, placement, weights, max_tokens_per_rank, rank=r, world=world, device=device,
                             _peers=peers)
    return layers


def call_all(layers, xs, outs=None, stream=None, skip=()):
    """One tg_moe_layer call of every virtual rank, as ONE launch; ranks in ``skip`` do not take
    part (a rank that died before the call).  Returns (status, outs); does not synchronise."""
    outs = outs or [torch.empty_like(x) for x in xs]
    xs2 = [None if r in skip else x for r, x in enumerate(xs)]
    rc = tg_moe_layer_multi([l.ctx for l in layers], xs2, outs, stream)
    return rc, outs


def failover_all(layers, xs, outs, stream=None, skip=()):
    """tg_failover of every virtual rank (except ``skip``), as one launch."""
    xs2 = [None if r in skip else x for r, x in enumerate(xs)]
    return tg_failover_multi([l.ctx for l in layers], xs2, outs, stream)
