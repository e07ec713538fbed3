"""NEXT-4: KV-segment checkpointing into the AW's checkpoint store between layer calls
(§6.1; segment size C = 2 H_kv (d / H_attn) S_elem = 4096 B per token and layer for
Mixtral, App. C), ordered commit records ("async log + commit") and
request-level restoration."""
import pytest
import torch

import workloads as wl

pytestmark = pytest.mark.gpu


def _kv_segment_bytes(d=4096, h_kv=8, h_attn=32, s_elem=2):
    return 2 * h_kv * (d // h_attn) * s_elem  # App. C


def test_segment_size_mixtral():
    assert _kv_segment_bytes() == 4096


def test_checkpoint_commit_restore_between_layer_calls():
    import paper_2601_01310_b200 as tg
    sh = wl.CONFIGS["tiny"]
    dev = torch.device("cuda", 0)
    pl = wl.make_placement(sh.E, 1, 1, shadows=False)
    L = wl.make_layer(sh, 5)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=sh.T, device=0)
    x = wl.make_tokens(sh, 5).to(dev)
    C = _kv_segment_bytes()
    steps, T = 12, sh.T
    seg_bytes = T * C
    tg.tg_kv_store_init(layer.ctx, steps * seg_bytes)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    segs = []
    for i in range(steps):
        layer(x)  # the layer call of this step; its KV segment is checkpointed after it
        seg = torch.randint(0, 256, (seg_bytes,), dtype=torch.uint8, device=dev, generator=g)
        segs.append(seg)
        tg.tg_kv_checkpoint(layer.ctx, seg, i * seg_bytes, i + 1)
    with pytest.raises(tg.TarragonError):  # sequence numbers must increase
        tg.tg_kv_checkpoint(layer.ctx, segs[0], 0, 3)
    with pytest.raises(tg.TarragonError):  # outside the bucket
        tg.tg_kv_checkpoint(layer.ctx, segs[0], steps * seg_bytes - 16, steps + 1)
    back = torch.empty(steps * seg_bytes, dtype=torch.uint8, device=dev)
    tg.tg_kv_restore(layer.ctx, back, 0)
    torch.cuda.synchronize()
    assert tg.tg_kv_committed(layer.ctx) == steps
    assert torch.equal(back, torch.cat(segs))
    # one request's segment alone (request-level restoration)
    one = torch.empty(seg_bytes, dtype=torch.uint8, device=dev)
    tg.tg_kv_restore(layer.ctx, one, 5 * seg_bytes)
    torch.cuda.synchronize()
    assert torch.equal(one, segs[5])
    layer.close()
