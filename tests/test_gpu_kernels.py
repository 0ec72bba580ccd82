"""Kernel-level parity on the B200: the tcgen05 GEMM and the paged attention against
plain PyTorch fp32 references of the same ops, plus the batch-invariance properties the
engine relies on (a row's result does not depend on which other rows share the launch).
"""

import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(W, X):
    import torch
    from paper_2603_13281_b200 import _lib
    lib = _lib.load()
    M, K = W.shape
    n = X.shape[0]
    out = torch.empty(n, M, dtype=torch.float32, device=W.device)
    _lib.check(lib.icr_gemm_bf16(W.data_ptr(), X.data_ptr(), out.data_ptr(), M, K, n,
                                 _lib.stream_handle()))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("M,K,n", [(128, 64, 16), (512, 256, 16), (4096, 4096, 16),
                                   (1024, 1024, 40), (256, 1024, 300), (6144, 4096, 16),
                                   (2048, 14336, 16)])
def test_gemm_matches_torch(cuda, M, K, n):
    import torch
    g = torch.Generator(device="cpu").manual_seed(M + K + n)
    W = (torch.randn(M, K, generator=g) / math.sqrt(K)).to(torch.bfloat16).to(cuda)
    X = torch.randn(n, K, generator=g).to(torch.bfloat16).to(cuda)
    got = _gemm(W, X)
    ref = X.float() @ W.float().T
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-4 * max(scale, 1.0) + 1e-4, (err, scale)


def test_gemm_row_result_independent_of_batch(cuda):
    """H1: a row computed in a 16-row launch equals the same row in a 256-row launch."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(7)
    M, K = 1024, 4096
    W = (torch.randn(M, K, generator=g) / 64).to(torch.bfloat16).to(cuda)
    X = torch.randn(256, K, generator=g).to(torch.bfloat16).to(cuda)
    big = _gemm(W, X)
    small = _gemm(W, X[:16].contiguous())
    mid = _gemm(W, X[:40].contiguous())
    assert torch.equal(big[:16], small)
    assert torch.equal(big[:40], mid)


def _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd):
    """fp32 restatement of layer_attention (src/model.py:384-425) over paged K/V."""
    import torch
    out = torch.zeros(q.shape[0], H * hd)
    G = H // Hkv
    for r in range(q.shape[0]):
        s, p = int(row_seq[r]), int(row_pos[r])
        pages = bt[s][: p // 16 + 1]
        K = torch.cat([kp[pg] for pg in pages], dim=1)[:, : p + 1].float()  # [Hkv, T, hd]
        V = torch.cat([vp[pg] for pg in pages], dim=1)[:, : p + 1].float()
        for h in range(H):
            g = h // G
            qs = q[r, h * hd:(h + 1) * hd].float()
            sc = (K[g] @ qs) * (1.0 / math.sqrt(hd))
            w = torch.softmax(sc, dim=0)
            out[r, h * hd:(h + 1) * hd] = w @ V[g]
    return out


def _run_attn(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd, chunk_pages):
    import torch
    from paper_2603_13281_b200 import _lib
    lib = _lib.load()
    out = torch.zeros_like(q)
    n_items = np.zeros(1, np.int32)
    bt_np = np.ascontiguousarray(bt, dtype=np.int32)
    rs = np.ascontiguousarray(row_seq, dtype=np.int32)
    rp = np.ascontiguousarray(row_pos, dtype=np.int32)
    _lib.check(lib.icr_paged_attention(
        q.data_ptr(), kp.data_ptr(), vp.data_ptr(), H, Hkv, hd, chunk_pages, q.shape[0],
        _lib.i32_ptr(rs), _lib.i32_ptr(rp), _lib.i32_ptr(bt_np), bt_np.shape[0], bt_np.shape[1],
        out.data_ptr(), _lib.i32_ptr(n_items), _lib.stream_handle()))
    return out, int(n_items[0])


@pytest.mark.parametrize("hd,H,Hkv", [(128, 32, 8), (64, 4, 2), (128, 2, 1)])
def test_paged_attention_matches_torch_and_sharing_is_bitwise(cuda, hd, H, Hkv):
    import torch
    g = torch.Generator(device="cpu").manual_seed(hd + H)
    n_pages = 64
    kp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    # 3 sequences: seqs 0,1 share 20 prefix pages (320 tokens), private tails; seq 2 private
    shared = list(range(0, 20))
    bt = np.full((3, 30), -1, np.int32)
    bt[0, :24] = shared + [20, 21, 22, 23]
    bt[1, :23] = shared + [24, 25, 26]
    bt[2, :10] = list(range(30, 40))
    row_seq = [0, 0, 1, 1, 2, 2]
    row_pos = [370, 370, 360, 360, 150, 150]
    q = torch.randn(len(row_seq), H * hd, generator=g).to(torch.bfloat16)
    ref = _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd)
    got, n_items = _run_attn(q.to(cuda), kp.to(cuda), vp.to(cuda), bt, row_seq, row_pos, H, Hkv,
                             hd, chunk_pages=4)
    err = (got.float().cpu() - ref).abs().max().item()
    assert err < 2e-2, err
    # Private copy of the shared prefix for seq 1 -> identical bytes out (layout invariance)
    kp2, vp2 = kp.clone(), vp.clone()
    kp2[40:60] = kp[0:20]
    vp2[40:60] = vp[0:20]
    bt2 = bt.copy()
    bt2[1, :20] = list(range(40, 60))
    got2, n_items2 = _run_attn(q.to(cuda), kp2.to(cuda), vp2.to(cuda), bt2, row_seq, row_pos, H,
                               Hkv, hd, chunk_pages=4)
    assert n_items2 > n_items  # sharing really merged work items
    assert torch.equal(got, got2)


@pytest.mark.parametrize("chunk_pages", [4, 8, 16, 32, 128])
def test_tc_attention_chunkings_match_torch(cuda, chunk_pages):
    """tcgen05 attention (head_dim 128) over 1..16 pipelined 8-page sub-chunks per item,
    partial last sub-chunks, private tails and a shared prefix, at every chunking the
    runtime exposes (chunk_pages is a deployment knob: 16 for decode, 128 for long context)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(7 + chunk_pages)
    H, Hkv, hd = 32, 8, 128
    shared = 45  # 720-token shared prefix: not a multiple of any sub-chunk
    n_pages = shared + 16
    kp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    n_seq = 4
    bt = np.full((n_seq, 50), -1, np.int32)
    for s in range(n_seq):
        bt[s, :shared] = np.arange(shared)
        bt[s, shared:shared + 2] = [shared + 2 * s, shared + 2 * s + 1]
    row_seq = [s for s in range(n_seq) for _ in range(2)]
    row_pos = [shared * 16 + 3 + s for s in range(n_seq) for _ in range(2)]
    # a few large-magnitude queries: the running max jumps between sub-chunks (O rescale path)
    q = torch.randn(len(row_seq), H * hd, generator=g)
    q[1::2] *= 3.0
    q = q.to(torch.bfloat16)
    ref = _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd)
    got, _ = _run_attn(q.to(cuda), kp.to(cuda), vp.to(cuda), bt, row_seq, row_pos, H, Hkv, hd,
                       chunk_pages=chunk_pages)
    err = (got.float().cpu() - ref).abs().max().item()
    assert err < 3e-2, err


@pytest.mark.parametrize("chunk_pages", [16, 64])
def test_tc_attention_workflow_shaped_prefill_and_decode(cuda, chunk_pages):
    """The C3 shape in miniature: many sequences on one long shared prefix (not a multiple of
    the chunk), each with private pages; prefill-style rows (consecutive positions, causal
    inside the last chunk, > 128 entries per chunk -> several items per chunk) and
    decode-style rows (encoder + decoder per sequence) in one launch."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(100 + chunk_pages)
    H, Hkv, hd = 32, 8, 128
    shared = 70  # 1120-token shared prefix
    n_seq = 12
    priv = 4
    n_pages = shared + n_seq * priv
    kp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    bt = np.full((n_seq, shared + priv), -1, np.int32)
    for s_ in range(n_seq):
        bt[s_, :shared] = np.arange(shared)
        bt[s_, shared:] = shared + priv * s_ + np.arange(priv)
    row_seq, row_pos = [], []
    for s_ in range(n_seq):
        if s_ % 3 == 0:  # prefill-style: 20 new rows after the prefix
            for i in range(20):
                row_seq.append(s_)
                row_pos.append(shared * 16 + i)
        else:  # decode-style: encoder + decoder row at one position
            for _ in range(2):
                row_seq.append(s_)
                row_pos.append(shared * 16 + 5 + s_)
    q = torch.randn(len(row_seq), H * hd, generator=g)
    q[1::2] *= 3.0
    q = q.to(torch.bfloat16)
    ref = _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd)
    got, _ = _run_attn(q.to(cuda), kp.to(cuda), vp.to(cuda), bt, row_seq, row_pos, H, Hkv, hd,
                       chunk_pages=chunk_pages)
    got = got.float().cpu()
    assert torch.isfinite(got).all()
    err = (got - ref).abs().max().item()
    assert err < 3e-2, err


def test_tc_attention_long_context_c4_shape(cuda):
    """C4 in miniature-free form: 16k shared context + a private page per sequence, 8
    sequences x (encoder, decoder) rows, 128-page chunks -> items of 16 pipelined sub-chunks
    (the regime where the epilogue once read O before the last P.V MMAs had finished). fp32
    torch reference on the device over the same bf16 K/V."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(21)
    H, Hkv, hd = 32, 8, 128
    shared, n_seq = 1024, 8
    n_pages = shared + n_seq
    kp = torch.randn(n_pages, Hkv, 16, hd, device="cuda", generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, device="cuda", generator=g).to(torch.bfloat16)
    bt = np.full((n_seq, shared + 1), -1, np.int32)
    for s_ in range(n_seq):
        bt[s_, :shared] = np.arange(shared)
        bt[s_, shared] = shared + s_
    row_seq = [s_ for s_ in range(n_seq) for _ in range(2)]
    row_pos = [shared * 16 + 3 + s_ for s_ in range(n_seq) for _ in range(2)]
    q = torch.randn(len(row_seq), H * hd, device="cuda", generator=g)
    q[1::2] *= 2.0
    q = q.to(torch.bfloat16)
    got, _ = _run_attn(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd, chunk_pages=128)
    # reference: [Hkv, T, hd] K/V of the shared prefix, plus each sequence's private page
    Kp = kp[:shared].float().permute(1, 0, 2, 3).reshape(Hkv, shared * 16, hd)
    Vp = vp[:shared].float().permute(1, 0, 2, 3).reshape(Hkv, shared * 16, hd)
    ref = torch.empty(len(row_seq), H * hd, device="cuda")
    for r, (s_, p_) in enumerate(zip(row_seq, row_pos)):
        tail = p_ - shared * 16 + 1
        K = torch.cat([Kp, kp[shared + s_].float()[:, :tail]], dim=1)
        V = torch.cat([Vp, vp[shared + s_].float()[:, :tail]], dim=1)
        qh = q[r].float().view(Hkv, H // Hkv, hd)
        w = torch.softmax(torch.einsum("gjd,gtd->gjt", qh, K) / math.sqrt(hd), dim=-1)
        ref[r] = torch.einsum("gjt,gtd->gjd", w, V).reshape(-1)
    err = (got.float() - ref).abs().max().item()
    assert torch.isfinite(got.float()).all() and err < 3e-2, err


def test_tc_attention_prefill_rows_causal_and_many_entries(cuda):
    """Prefill-shaped work: 48 rows of one sequence at consecutive positions (causal mask
    inside the chunk, rows sharing pages at different positions), 48 x 4 heads = 192 query
    entries per KV head -> more than one 128-entry item per chunk."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(11)
    H, Hkv, hd = 32, 8, 128
    n_pages = 12
    kp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    bt = np.full((1, 16), -1, np.int32)
    bt[0, :n_pages] = np.arange(n_pages)
    row_pos = list(range(130, 178))
    row_seq = [0] * len(row_pos)
    q = torch.randn(len(row_seq), H * hd, generator=g).to(torch.bfloat16)
    ref = _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd)
    for chunk_pages in (8, 16):
        got, n_items = _run_attn(q.to(cuda), kp.to(cuda), vp.to(cuda), bt, row_seq, row_pos, H, Hkv,
                                 hd, chunk_pages=chunk_pages)
        err = (got.float().cpu() - ref).abs().max().item()
        assert err < 2e-2, (chunk_pages, err)


def test_tc_attention_narrow_and_wide_items_are_bitwise_equal(cuda):
    """Items with <= 64 query entries run the 16-lane softmax form, wider items the 32-lane
    form; a row's output must not depend on which form served it (batch invariance): 20
    sequences on one shared prefix (160 entries per KV head -> a 128-entry wide item plus a
    narrow one per chunk) against every sequence run alone (8 entries: narrow). Positions
    differ per sequence so causal edges cut sub-chunks, and some queries are scaled up so the
    running max moves between sub-chunks (O rescale path)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(5)
    H, Hkv, hd = 32, 8, 128
    shared, n_seq, priv = 37, 20, 2
    n_pages = shared + n_seq * priv
    kp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    vp = torch.randn(n_pages, Hkv, 16, hd, generator=g).to(torch.bfloat16)
    bt = np.full((n_seq, shared + priv), -1, np.int32)
    for s_ in range(n_seq):
        bt[s_, :shared] = np.arange(shared)
        bt[s_, shared:] = shared + priv * s_ + np.arange(priv)
    row_seq = [s_ for s_ in range(n_seq) for _ in range(2)]
    row_pos = [shared * 16 + 1 + s_ for s_ in range(n_seq) for _ in range(2)]
    q = torch.randn(len(row_seq), H * hd, generator=g)
    q[1::4] *= 4.0
    q = q.to(torch.bfloat16)
    kd, vd = kp.to(cuda), vp.to(cuda)
    for chunk_pages in (8, 16, 64):
        together, n_items = _run_attn(q.to(cuda), kd, vd, bt, row_seq, row_pos, H, Hkv, hd,
                                      chunk_pages=chunk_pages)
        for s_ in range(n_seq):
            alone, _ = _run_attn(q[2 * s_:2 * s_ + 2].to(cuda), kd, vd, bt[s_:s_ + 1], [0, 0],
                                 row_pos[2 * s_:2 * s_ + 2], H, Hkv, hd, chunk_pages=chunk_pages)
            assert torch.equal(together[2 * s_:2 * s_ + 2], alone), (chunk_pages, s_)
    ref = _attention_ref(q, kp, vp, bt, row_seq, row_pos, H, Hkv, hd)
    err = (together.float().cpu() - ref).abs().max().item()
    assert err < 3e-2, err
