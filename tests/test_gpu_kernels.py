"""Kernel-level parity on the B200, through the C-ABI library.

Integer work (policy, compaction, gathers) is bit-exact against the oracle
and the reference golden vectors; tensor-core work is compared with a plain
PyTorch fp32 reference of the same op on the same bf16 inputs.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import selection as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def dev():
    from paper_2310_18481_b200 import build, device
    build.build()
    device.lib()
    return device


def test_policy_select_bit_exact_vs_reference_golden(dev):
    cases = json.loads((GOLDEN / "policy_cases.json").read_text())
    # group by (dispatch, factor) so each launch has one scalar pair
    groups = {}
    for c in cases:
        groups.setdefault((c["dispatch_us"], c["factor"]), []).append(c)
    mismatches = 0
    for (dispatch, factor), cs in groups.items():
        width = max(len(c["lat_us"]) for c in cs)
        lat = np.zeros((len(cs), width), dtype=np.int64)
        cr = np.zeros((len(cs), width), dtype=np.int32)
        for i, c in enumerate(cs):
            lat[i, : len(c["lat_us"])] = c["lat_us"]
            cr[i, : len(c["credit"])] = c["credit"]
        ncand = np.array([len(c["lat_us"]) for c in cs], dtype=np.int32)
        dl = np.array([c["deadline_us"] for c in cs], dtype=np.int64)
        got = dev.policy_select(lat, cr, ncand, dl, dispatch, factor)
        exp = np.array([c["expected"] for c in cs], dtype=np.int32)
        mismatches += int((got != exp).sum())
    assert mismatches == 0, f"{mismatches} of {len(cases)} policy choices differ from the reference"


def test_policy_select_batched_random_vs_oracle(dev):
    rng = np.random.default_rng(3)
    n, width = 4096, 40  # > 32 candidates exercises the multi-round warp path
    lat = np.sort(rng.integers(1_000, 400_000, size=(n, width)), axis=1).astype(np.int64)
    lat += np.arange(width)  # strictly increasing
    ncand = rng.integers(0, width + 1, size=n).astype(np.int32)
    dl = rng.integers(-5_000, 500_000, size=n).astype(np.int64)
    for factor in (0.5, 1.0, 1.37, 2.5):
        got = dev.policy_select(lat, None, ncand, dl, 0, factor)
        exp = orc.policy_select(lat, ncand, dl, 0, factor)
        assert np.array_equal(got, exp)


@pytest.mark.parametrize("n,k", [(0, 3), (1, 1), (7, 2), (256, 3), (1000, 4), (1025, 3), (3000, 4), (517, 8)])
def test_compact_index_bit_exact(dev, n, k):
    rng = np.random.default_rng(n * 31 + k)
    masks = rng.integers(1, 1 << k, size=n).astype(np.int64)
    m_dev = torch.as_tensor(masks.astype(np.int16)).cuda()
    idx, inv, counts, offs, perm = dev.compact_index(m_dev, k)
    e_idx, e_inv, e_counts = orc.compact(masks, k)
    assert counts.cpu().numpy().tolist() == e_counts.tolist()
    for kk in range(k):
        c = int(e_counts[kk])
        assert np.array_equal(idx[kk, :c].cpu().numpy(), e_idx[kk])
        assert np.array_equal(inv[kk].cpu().numpy(), e_inv[kk])
    e_perm, e_offs, _ = orc.group_free_masks(masks if n else np.zeros(0, np.int64), 4)
    if n:
        bins = 1 << k
        ref_perm = np.argsort(masks, kind="stable")
        ref_offs = np.concatenate([[0], np.cumsum(np.bincount(masks, minlength=bins))])
        assert np.array_equal(perm.cpu().numpy(), ref_perm)
        assert np.array_equal(offs.cpu().numpy(), ref_offs)


def test_gather_rows_with_slots(dev):
    rng = np.random.default_rng(0)
    pool = torch.randn(50, 3, 40, dtype=torch.float32, device="cuda").to(torch.bfloat16)
    idx = torch.tensor([3, 1, 4, 1, 5], dtype=torch.int32, device="cuda")
    slot = torch.as_tensor(rng.permutation(50).astype(np.int32)).cuda()
    count = torch.tensor([4], dtype=torch.int32, device="cuda")
    dst = torch.zeros(5, 3, 40, dtype=torch.bfloat16, device="cuda")
    dev.gather_rows(pool, idx, count, 5, dst, slot=slot)
    torch.cuda.synchronize()
    exp = pool[slot[idx[:4].long()].long()]
    assert torch.equal(dst[:4], exp)
    assert torch.equal(dst[4], torch.zeros_like(dst[4]))


def _bf(t):
    return t.to(torch.bfloat16)


def _close(got, ref, tol=2e-2):
    err = (got.float() - ref.float()).abs().max().item()
    scale = ref.float().abs().max().item() + 1e-6
    return err <= tol * scale, err, scale


@pytest.mark.parametrize("M,K,N,BN,relu", [
    (128, 64, 64, 64, False), (1, 64, 32, 32, False), (300, 192, 96, 96, True),
    (1000, 1024, 256, 256, True), (517, 576, 352, 192, True), (64, 3072, 512, 128, True),
])
def test_gemm_dense_vs_torch(dev, M, K, N, BN, relu):
    g = torch.Generator(device="cpu").manual_seed(M + K + N)
    A = _bf(torch.randn(M, K, generator=g)).cuda()
    Kp = (K + 63) // 64 * 64
    W = torch.zeros(N, Kp, dtype=torch.bfloat16)
    W[:, :K] = _bf(torch.randn(N, K, generator=g) * 0.05)
    W = W.cuda()
    b = (torch.randn(N, generator=g) * 0.1).cuda()
    D = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_dense(A, W, b, D, BN=BN, relu=relu)
    p.run()
    torch.cuda.synchronize()
    ref = A.float().cpu() @ W[:, :K].float().cpu().T + b.cpu()
    if relu:
        ref = ref.clamp_min(0)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


def test_gemm_dense_fp32_out_and_segments(dev):
    g = torch.Generator().manual_seed(7)
    M, K = 200, 256
    A = _bf(torch.randn(M, K, generator=g)).cuda()
    W = _bf(torch.randn(160, K, generator=g) * 0.05).cuda()
    D1 = torch.zeros(M, 96, dtype=torch.bfloat16, device="cuda")
    D2 = torch.zeros(M, 200, dtype=torch.bfloat16, device="cuda")
    segs = [(0, 64, D1, 96, 32), (64, 160, D2, 200, 104)]
    p = dev.plan_dense(A, W, None, D1, BN=160, segs=segs)
    p.run()
    L = torch.zeros(M, 397, dtype=torch.float32, device="cuda")
    W2 = _bf(torch.randn(397, K, generator=g) * 0.05).cuda()
    dev.plan_dense(A, W2, None, L, BN=128, out_fp32=True).run()
    torch.cuda.synchronize()
    ref = A.float().cpu() @ W.float().cpu().T
    assert _close(D1[:, 32:96].cpu(), ref[:, :64])[0]
    assert _close(D2[:, 104:200].cpu(), ref[:, 64:160])[0]
    assert torch.count_nonzero(D1[:, :32]) == 0
    ref2 = A.float().cpu() @ W2.float().cpu().T
    assert _close(L.cpu(), ref2, tol=1e-3)[0]


def _conv_weights(Cout, Cin, k, g):
    w = _bf(torch.randn(Cout, Cin, k, k, generator=g) * (2.0 / (Cin * k * k)) ** 0.5)
    cc = (Cin + 63) // 64
    packed = torch.zeros(Cout, k * k, cc * 64, dtype=torch.bfloat16)
    packed[:, :, :Cin] = w.permute(0, 2, 3, 1).reshape(Cout, k * k, Cin)
    return w, packed.reshape(Cout, -1).contiguous()


@pytest.mark.parametrize("n,H,Cin,Cout,k,s,pad,tile,BN", [
    (2, 14, 64, 96, 3, 1, 1, (1, 7, 14), 96),
    (3, 28, 96, 96, 3, 2, 1, (1, 7, 14), 96),
    (5, 7, 160, 224, 3, 1, 1, (2, 7, 7), 224),
    (4, 56, 64, 192, 3, 1, 1, (1, 8, 16), 192),
    (2, 8, 192, 320, 3, 1, 1, (2, 8, 8), 160),
    (2, 28, 320, 160, 3, 2, 1, (1, 7, 14), 160),
])
def test_conv_implicit_gemm_vs_torch(dev, n, H, Cin, Cout, k, s, pad, tile, BN):
    g = torch.Generator().manual_seed(n * H + Cin)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, k, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    OH = (H + 2 * pad - k) // s + 1
    D = torch.zeros(n * OH * OH, Cout, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X, n, H, H, Cin, Cin, k, k, s, pad, packed.cuda(), Cout, b.cuda(), D, ldd=Cout,
                      BN=BN, relu=True, tile=tile)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=s, padding=pad).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin,Cout,s,split", [
    (5, 7, 160, 224, 1, 1), (5, 7, 160, 224, 1, 3), (3, 14, 192, 320, 2, 4), (2, 8, 224, 224, 1, 6),
])
def test_conv_split_k_into_concat_slice(dev, n, H, Cin, Cout, s, split):
    """Split-K implicit-GEMM conv (fp32 workspace + finalize) writing a
    channel slice of a wider concat output, as the Inception branches do; run
    twice (the finalize re-zeroes the workspace)."""
    g = torch.Generator().manual_seed(n * H + Cin + split)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, 3, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    OH = (H + 2 - 3) // s + 1
    ldd, col0 = Cout + 96, 64
    D = torch.full((n * OH * OH, ldd), 7.0, dtype=torch.bfloat16, device="cuda")
    from paper_2310_18481_b200.encoders import pick_bn, pick_conv_tile
    p = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, s, 1, packed.cuda(), Cout, b.cuda(), D, ldd=ldd, col0=col0,
                      BN=pick_bn(Cout), relu=True, tile=pick_conv_tile(n, OH, OH), split_k=split)
    assert getattr(p, "split_k", 1) == split
    p.run()
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=s, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D[:, col0:col0 + Cout].cpu(), ref)
    assert ok, (err, scale)
    assert torch.all(D[:, :col0] == 7.0) and torch.all(D[:, col0 + Cout:] == 7.0)  # neighbours untouched


def test_gather_concat_gemm_vs_torch(dev):
    g = torch.Generator().manual_seed(11)
    N, F, K = 300, 1024, 3
    masks = torch.randint(1, 8, (N,), generator=g)
    feats, invs = [], []
    full = torch.zeros(N, K * F)
    for k in range(K):
        have = ((masks >> k) & 1).bool()
        nk = int(have.sum())
        f = _bf(torch.randn(nk, F, generator=g))
        inv = torch.full((N,), -1, dtype=torch.int32)
        inv[have] = torch.arange(nk, dtype=torch.int32)
        full[have, k * F:(k + 1) * F] = f.float()
        feats.append(f.cuda())
        invs.append(inv)
    inv = torch.stack(invs).cuda()
    W = _bf(torch.randn(512, K * F, generator=g) * 0.02)
    b = torch.randn(512, generator=g) * 0.1
    H = torch.zeros(N, 512, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_gather(feats, inv, W.cuda(), b.cuda(), H, M=N, feat_dim=F, BN=256, relu=True)
    p.run()
    torch.cuda.synchronize()
    ref = (full @ W.float().T + b).clamp_min(0)
    ok, err, scale = _close(H.cpu(), ref)
    assert ok, (err, scale)


def test_pool_im2col_segment_mean(dev):
    L = dev.lib()
    g = torch.Generator().manual_seed(5)
    x = _bf(torch.randn(3, 64, 28, 28, generator=g))
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    # max 3x3 s2 ceil -> 14x14 written into a 96-wide concat slice at col 32
    Y = torch.zeros(3 * 14 * 14, 96, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_pool2d(dev.ptr(X), 3, 28, 28, 64, 64, 3, 2, 0, 1, 1, dev.ptr(Y), 96, 32, dev.stream_ptr()), "pool")
    ref = torch.nn.functional.max_pool2d(x.float(), 3, 2, 0, ceil_mode=True).permute(0, 2, 3, 1).reshape(-1, 64)
    torch.cuda.synchronize()
    assert torch.equal(Y[:, 32:].cpu().float(), ref)
    # avg 3x3 s1 p1 (count_include_pad)
    Z = torch.zeros(3 * 28 * 28, 64, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_pool2d(dev.ptr(X), 3, 28, 28, 64, 64, 3, 1, 1, 0, 0, dev.ptr(Z), 64, 0, dev.stream_ptr()), "pool")
    ref = torch.nn.functional.avg_pool2d(x.float(), 3, 1, 1).permute(0, 2, 3, 1).reshape(-1, 64)
    torch.cuda.synchronize()
    assert _close(Z.cpu(), ref, tol=1e-2)[0]
    # im2col of a 3-channel 7x7/2 conv
    xi = _bf(torch.randn(2, 3, 32, 32, generator=g))
    Xi = xi.permute(0, 2, 3, 1).contiguous().cuda()
    out = torch.zeros(2 * 16 * 16, 192, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_im2col(dev.ptr(Xi), 2, 32, 32, 3, 7, 7, 2, 3, dev.ptr(out), 192, dev.stream_ptr()), "im2col")
    cols = torch.nn.functional.unfold(xi.float(), 7, padding=3, stride=2)  # [n, C*49, L] (c, kh, kw)
    cols = cols.reshape(2, 3, 49, 256).permute(0, 3, 2, 1).reshape(2 * 256, 147)
    torch.cuda.synchronize()
    assert torch.equal(out[:, :147].cpu().float(), cols)
    assert torch.count_nonzero(out[:, 147:]) == 0
    # segment mean
    f = _bf(torch.randn(4 * 3 * 49, 64, generator=g)).cuda()
    y = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_segment_mean(dev.ptr(f), 4, 3, 49, 64, dev.ptr(y), 64, dev.stream_ptr()), "segmean")
    torch.cuda.synchronize()
    ref = f.float().cpu().reshape(4, 147, 64).mean(1)
    assert _close(y.cpu(), ref, tol=1e-2)[0]


@pytest.mark.parametrize("n,H,Cin,Cpad,tile", [
    (2, 32, 3, 8, (1, 8, 16)), (3, 64, 10, 16, (1, 8, 16)), (2, 64, 1, 8, (1, 4, 32)),
    (5, 224, 3, 8, (1, 8, 16)),
])
def test_conv_small_channel_direct_vs_torch(dev, n, H, Cin, Cpad, tile):
    """7x7/2 first-layer conv read straight from channel-padded, W-padded NHWC
    frames (MODE_CONV_SMALLC: one overlapping-stride 5-D TMA box per K block)."""
    from paper_2310_18481_b200.encoders import pack_smallc_weight
    g = torch.Generator().manual_seed(H + Cin)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    X = torch.zeros(n, H, H + 6, Cpad, dtype=torch.bfloat16)  # W pre-padded by 3 per side
    X[:, :, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
    OH = (H + 6 - 7) // 2 + 1
    D = torch.zeros(n * OH * OH, 64, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X.cuda(), n, H, H, Cpad, Cpad, 7, 7, 2, 3, pack_smallc_weight(w, Cpad).cuda(), 64,
                      b.cuda(), D, ldd=64, BN=64, relu=True, tile=tile)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=2, padding=3).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, 64)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("c_src,c_dst,pad_w", [(3, 8, 3), (10, 16, 3), (1, 8, 0), (16, 16, 2)])
def test_gather_rows_channel_and_line_pad(dev, c_src, c_dst, pad_w):
    L = dev.lib()
    lines, width = 3 * 17, 19
    pool = _bf(torch.randn(9, lines, width, c_src)).cuda()
    idx = torch.tensor([4, 0, 7], dtype=torch.int32, device="cuda")
    slot = torch.tensor([8, 7, 6, 5, 4, 3, 2, 1, 0], dtype=torch.int32, device="cuda")
    count = torch.tensor([3], dtype=torch.int32, device="cuda")
    dst = torch.full((3, lines, width + 2 * pad_w, c_dst), 7.0, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_gather_rows_pad(dev.ptr(pool), lines, width, c_src, c_dst, pad_w, dev.ptr(slot),
                                   dev.ptr(idx), dev.ptr(count), 3, dev.ptr(dst), dev.stream_ptr()), "gather_pad")
    torch.cuda.synchronize()
    src = pool[slot[idx.long()].long()]
    assert torch.equal(dst[:, :, pad_w:pad_w + width, :c_src], src)
    dst[:, :, pad_w:pad_w + width, :c_src] = 0
    assert torch.count_nonzero(dst) == 0


@pytest.mark.parametrize("M,K,N,BN,split,act", [
    (48, 3072, 512, 256, 12, 1), (1, 768, 2304, 256, 3, 0), (197, 3072, 768, 256, 8, 0), (40, 768, 3129, 224, 4, 0),
])
def test_gemm_split_k_vs_torch(dev, M, K, N, BN, split, act):
    g = torch.Generator().manual_seed(M * 7 + N)
    A = _bf(torch.randn(M, K, generator=g)).cuda()
    W = _bf(torch.randn(N, K, generator=g) * 0.03).cuda()
    b = (torch.randn(N, generator=g) * 0.1).cuda()
    out_fp32 = N == 3129
    D = torch.zeros(M, N, dtype=torch.float32 if out_fp32 else torch.bfloat16, device="cuda")
    R = _bf(torch.randn(M, N, generator=g)).cuda() if (N == 768 and not out_fp32) else None
    if R is not None:
        D.copy_(R)
    p = dev.plan_dense(A, W, b, D, BN=BN, act=act, out_fp32=out_fp32, split_k=split,
                       residual=D if R is not None else None)
    assert p.split_k == split
    p.run()
    p.run()  # the workspace is re-zeroed every run
    torch.cuda.synchronize()
    ref = A.float().cpu() @ W.float().cpu().T + b.cpu()
    if act == 1:
        ref = ref.clamp_min(0)
    if R is not None:  # residual applied twice (in-place D += ...)
        ref = R.float().cpu() + 2 * ref
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


def test_gather_gemm_split_k(dev):
    g = torch.Generator().manual_seed(5)
    N_req, F, K = 37, 1024, 3
    masks = torch.randint(1, 8, (N_req,), generator=g)
    feats, invs = [], []
    full = torch.zeros(N_req, K * F)
    for k in range(K):
        have = ((masks >> k) & 1).bool()
        f = _bf(torch.randn(int(have.sum()), F, generator=g))
        inv = torch.full((N_req,), -1, dtype=torch.int32)
        inv[have] = torch.arange(int(have.sum()), dtype=torch.int32)
        full[have, k * F:(k + 1) * F] = f.float()
        feats.append(f.cuda())
        invs.append(inv)
    W = _bf(torch.randn(512, K * F, generator=g) * 0.02)
    b = torch.randn(512, generator=g) * 0.1
    H = torch.zeros(N_req, 512, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_gather(feats, torch.stack(invs).cuda(), W.cuda(), b.cuda(), H, M=N_req, feat_dim=F, BN=256,
                        relu=True, split_k=6)
    assert p.split_k == 6
    p.run()
    torch.cuda.synchronize()
    ref = (full @ W.float().T + b).clamp_min(0)
    ok, err, scale = _close(H.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("c_src,c_dst,u8,width", [(3, 8, True, 224), (10, 16, True, 224), (1, 8, False, 256),
                                                   (3, 8, False, 40)])
def test_gather_staged_lines_u8_and_bf16(dev, c_src, c_dst, u8, width):
    """Line-staged (smem, 16-B vector) padding gather; uint8 pools are
    converted to bf16 as u8 * scale + bias."""
    import ctypes
    L = dev.lib()
    lines, pad = 6, 3
    if u8:
        pool = torch.randint(0, 256, (5, lines, width, c_src), dtype=torch.uint8).cuda()
        ref_pool = (pool.float() / 64.0 - 2.0).to(torch.bfloat16)
    else:
        pool = _bf(torch.randn(5, lines, width, c_src)).cuda()
        ref_pool = pool
    idx = torch.tensor([3, 0, 4], dtype=torch.int32, device="cuda")
    cnt = torch.tensor([3], dtype=torch.int32, device="cuda")
    dst = torch.full((3, lines, width + 2 * pad, c_dst), 5.0, dtype=torch.bfloat16, device="cuda")
    rows = (dev.RowDesc * 1)(dev.RowDesc(lines, width, c_src, c_dst, pad, int(u8), 1.0 / 64.0, -2.0))
    mask = torch.ones(5, dtype=torch.int16, device="cuda")  # every request has modality 0
    mask[1] = 0
    mask[2] = 0
    X = (ctypes.c_void_p * 1)(pool.data_ptr())
    G = (ctypes.c_void_p * 1)(dst.data_ptr())
    ix = torch.empty(5, dtype=torch.int32, device="cuda")
    inv = torch.empty(5, dtype=torch.int32, device="cuda")
    offs = torch.empty(3, dtype=torch.int32, device="cuda")
    perm = torch.empty(5, dtype=torch.int32, device="cuda")
    dev.check(L.ms_compact(mask.data_ptr(), 5, 1, X, rows, None, G, ix.data_ptr(), inv.data_ptr(),
                           cnt.data_ptr(), offs.data_ptr(), perm.data_ptr(), dev.stream_ptr()), "compact")
    torch.cuda.synchronize()
    assert ix[:3].cpu().tolist() == [0, 3, 4]
    exp = ref_pool[torch.tensor([0, 3, 4]).cuda()]
    assert torch.equal(dst[:, :, pad:pad + width, :c_src], exp)
    dst[:, :, pad:pad + width, :c_src] = 0
    assert torch.count_nonzero(dst) == 0


@pytest.mark.parametrize("c_src,u8,width", [(3, True, 224), (1, False, 256), (3, False, 40)])
def test_gather_four_channel_frames_with_row_padding(dev, c_src, u8, width):
    """4-channel (8-byte) destination pixels with frame row padding
    (MsRowDesc frame_h/pad_h): each frame's rows land between pad_h rows the
    gather never writes, W-pad columns and the pad channel are zeroed."""
    import ctypes
    L = dev.lib()
    frames, fh, pad, pad_h = 2, 3, 3, 2
    lines = frames * fh
    if u8:
        pool = torch.randint(0, 256, (5, lines, width, c_src), dtype=torch.uint8).cuda()
        ref_pool = (pool.float() / 64.0 - 2.0).to(torch.bfloat16)
    else:
        pool = _bf(torch.randn(5, lines, width, c_src)).cuda()
        ref_pool = pool
    cnt = torch.tensor([3], dtype=torch.int32, device="cuda")
    dst = torch.full((3, frames, fh + 2 * pad_h, width + 2 * pad, 4), 5.0, dtype=torch.bfloat16, device="cuda")
    rows = (dev.RowDesc * 1)(dev.RowDesc(lines, width, c_src, 4, pad, int(u8), 1.0 / 64.0, -2.0, fh, pad_h))
    mask = torch.ones(5, dtype=torch.int16, device="cuda")
    mask[1] = 0
    mask[2] = 0
    X = (ctypes.c_void_p * 1)(pool.data_ptr())
    G = (ctypes.c_void_p * 1)(dst.data_ptr())
    ix = torch.empty(5, dtype=torch.int32, device="cuda")
    inv = torch.empty(5, dtype=torch.int32, device="cuda")
    offs = torch.empty(3, dtype=torch.int32, device="cuda")
    perm = torch.empty(5, dtype=torch.int32, device="cuda")
    dev.check(L.ms_compact(mask.data_ptr(), 5, 1, X, rows, None, G, ix.data_ptr(), inv.data_ptr(),
                           cnt.data_ptr(), offs.data_ptr(), perm.data_ptr(), dev.stream_ptr()), "compact")
    torch.cuda.synchronize()
    exp = ref_pool[torch.tensor([0, 3, 4]).cuda()].view(3, frames, fh, width, c_src)
    body = dst[:, :, pad_h:pad_h + fh]
    assert torch.equal(body[:, :, :, pad:pad + width, :c_src], exp)
    body[:, :, :, pad:pad + width, :c_src] = 0
    assert torch.count_nonzero(body) == 0  # W-pad columns and pad channels zeroed
    assert torch.all(dst[:, :, :pad_h] == 5.0) and torch.all(dst[:, :, pad_h + fh:] == 5.0)  # pad rows untouched


@pytest.mark.parametrize("n,H,Cin,tile", [(2, 32, 10, (1, 8, 16)), (3, 224, 10, (1, 8, 16)), (2, 64, 12, (1, 4, 32))])
def test_conv_twelve_channel_row_padded_vs_torch(dev, n, H, Cin, tile):
    """7x7/2 first-layer conv over 12-channel row+column padded frames (flow:
    MODE_CONV_C12, three 32-element SW64 parts per filter row)."""
    from paper_2310_18481_b200.encoders import pack_c12_weight
    g = torch.Generator().manual_seed(H + Cin + 17)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    X = torch.zeros(n, H + 6, H + 6, 12, dtype=torch.bfloat16)
    X[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
    OH = (H + 6 - 7) // 2 + 1
    D = torch.zeros(n * OH * OH, 64, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X.cuda(), n, H, H, 12, 12, 7, 7, 2, 3, pack_c12_weight(w).cuda(), 64,
                      b.cuda(), D, ldd=64, BN=64, relu=True, tile=tile)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=2, padding=3).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, 64)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin,tile", [(2, 32, 3, (1, 8, 16)), (2, 64, 1, (1, 4, 32)), (5, 224, 3, (1, 8, 16)),
                                          (3, 256, 1, (1, 8, 16))])
def test_conv_four_channel_row_padded_vs_torch(dev, n, H, Cin, tile):
    """7x7/2 first-layer conv over 4-channel, row- and column-padded frames
    (MODE_CONV_C4: 5-D TMA, one 128-B K block per filter-row pair)."""
    from paper_2310_18481_b200.encoders import pack_c4_weight
    g = torch.Generator().manual_seed(H + Cin + 7)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    X = torch.zeros(n, H + 6, H + 6, 4, dtype=torch.bfloat16)
    X[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
    OH = (H + 6 - 7) // 2 + 1
    D = torch.zeros(n * OH * OH, 64, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X.cuda(), n, H, H, 4, 4, 7, 7, 2, 3, pack_c4_weight(w).cuda(), 64,
                      b.cuda(), D, ldd=64, BN=64, relu=True, tile=tile)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=2, padding=3).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, 64)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin", [(2, 32, 3), (2, 64, 1), (3, 30, 3), (5, 224, 3), (3, 256, 1), (1, 224, 3)])
def test_stem_conv_pool_fused_vs_unfused_and_torch(dev, n, H, Cin):
    """MODE_STEM_POOL: 7x7/2 conv (raw padded rows as no-swizzle UMMA
    operands) + ReLU + 3x3/2 ceil max pool in one kernel == the C4 conv
    kernel followed by the pool, and == torch within bf16 tolerance."""
    from paper_2310_18481_b200.encoders import pack_c4_weight, pack_stem_weight
    g = torch.Generator().manual_seed(H + Cin + 11)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    X = torch.zeros(n, H + 6, H + 6, 4, dtype=torch.bfloat16)
    X[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
    Xd, Wd, bd = X.cuda(), pack_c4_weight(w).cuda(), b.cuda()
    OH = (H + 6 - 7) // 2 + 1
    PH = -(-(OH - 3) // 2) + 1
    Y = torch.full((n * PH * PH, 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    dev.plan_stem_pool(Xd, n, H, H, 7, 3, pack_stem_weight(w).cuda(), bd, Y, ldy=64).run()
    D = torch.zeros(n * OH * OH, 64, dtype=torch.bfloat16, device="cuda")
    dev.plan_conv(Xd, n, H, H, 4, 4, 7, 7, 2, 3, Wd, 64, bd, D, ldd=64, BN=64, relu=True, tile=(1, 8, 16)).run()
    torch.cuda.synchronize()
    pooled = torch.nn.functional.max_pool2d(D.float().reshape(n, OH, OH, 64).permute(0, 3, 1, 2), 3, 2,
                                            ceil_mode=True)
    pooled = pooled.permute(0, 2, 3, 1).reshape(-1, 64)
    assert torch.isfinite(Y.float()).all()
    # same bf16 conv values, max is exact: allow one bf16 ulp for accumulation order
    diff = (Y.float().cpu() - pooled.cpu()).abs()
    assert float((diff > pooled.cpu().abs() * 2 ** -7 + 1e-6).float().mean()) == 0.0, float(diff.max())
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=2, padding=3).clamp_min(0)
    ref = torch.nn.functional.max_pool2d(ref, 3, 2, ceil_mode=True).permute(0, 2, 3, 1).reshape(-1, 64)
    ok, err, scale = _close(Y.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin", [(2, 32, 10), (3, 224, 10), (2, 64, 12)])
def test_stem_conv_pool_three_planes_vs_torch(dev, n, H, Cin):
    """MODE_STEM_POOL over three 4-channel planes (flow's 10 channels padded
    to 12): same fused conv + ReLU + max pool, planar input layout."""
    from paper_2310_18481_b200.encoders import pack_stem_weight_planes
    g = torch.Generator().manual_seed(H + Cin + 17)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    Hp = H + 6
    X = torch.zeros(3, n, Hp, Hp, 4, dtype=torch.bfloat16)
    xp = torch.zeros(n, Hp, Hp, 12, dtype=torch.bfloat16)
    xp[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
    for q in range(3):
        X[q] = xp[..., 4 * q:4 * q + 4]
    OH = (H + 6 - 7) // 2 + 1
    PH = -(-(OH - 3) // 2) + 1
    Y = torch.full((n * PH * PH, 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    dev.plan_stem_pool(X.cuda(), n, H, H, 7, 3, pack_stem_weight_planes(w).cuda(), b.cuda(), Y, ldy=64, planes=3,
                       plane_stride=n * Hp * Hp * 4).run()
    torch.cuda.synchronize()
    assert torch.isfinite(Y.float()).all()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=2, padding=3).clamp_min(0)
    ref = torch.nn.functional.max_pool2d(ref, 3, 2, ceil_mode=True).permute(0, 2, 3, 1).reshape(-1, 64)
    ok, err, scale = _close(Y.cpu(), ref)
    assert ok, (err, scale)


def test_gather_planar_twelve_channels(dev):
    """ms_compact's planar 12-channel gather (plane q = channels 4q..4q+3) ==
    the interleaved gather split into planes."""
    torch.manual_seed(5)
    N, S, Hs, Ws, C = 3, 2, 6, 16, 10
    pool = torch.randint(0, 256, (4, S, Hs, Ws, C), dtype=torch.uint8, device="cuda")
    mask = torch.tensor([1, 1, 1], dtype=torch.int16, device="cuda")
    slot = torch.tensor([2, 0, 3], dtype=torch.int32, device="cuda")
    pad, ph = 3, 3
    Hp, Wp = Hs + 2 * ph, Ws + 2 * pad
    outs = []
    for planar in (False, True):
        G = torch.zeros(N * S * Hp * Wp * 12, dtype=torch.bfloat16, device="cuda")
        stride = N * S * Hp * Wp * 4 if planar else 0
        rows = (dev.RowDesc * 1)(dev.RowDesc(S * Hs, Ws, C, 12, pad, 1, 1.0 / 64.0, -2.0, Hs, ph, 0, stride))
        idx = torch.zeros(N, dtype=torch.int32, device="cuda")
        inv = torch.zeros(N, dtype=torch.int32, device="cuda")
        counts = torch.zeros(1, dtype=torch.int32, device="cuda")
        offs = torch.zeros(3, dtype=torch.int32, device="cuda")
        perm = torch.zeros(N, dtype=torch.int32, device="cuda")
        import ctypes
        Xp = (ctypes.c_void_p * 1)(pool.data_ptr())
        Gp = (ctypes.c_void_p * 1)(G.data_ptr())
        dev.check(dev.lib().ms_compact(mask.data_ptr(), N, 1, Xp, rows, slot.data_ptr(), Gp, idx.data_ptr(),
                                       inv.data_ptr(), counts.data_ptr(), offs.data_ptr(), perm.data_ptr(),
                                       dev.stream_ptr()), "ms_compact")
        torch.cuda.synchronize()
        outs.append(G.cpu())
    inter = outs[0].reshape(N * S, Hp, Wp, 12)
    planar = outs[1].reshape(3, N * S, Hp, Wp, 4)
    for q in range(3):
        assert torch.equal(planar[q], inter[..., 4 * q:4 * q + 4])


@pytest.mark.parametrize("M,K,N,BN", [(1000, 1024, 256, 256), (300, 192, 96, 96), (128, 64, 64, 64), (517, 576, 352, 192)])
def test_gemm_cta_pair_dense_vs_torch(dev, M, K, N, BN):
    """2-CTA clusters (tcgen05.mma.cta_group::2, M=256 tiles)."""
    g = torch.Generator().manual_seed(M + 3 * N)
    A = _bf(torch.randn(M, K, generator=g)).cuda()
    W = _bf(torch.randn(N, K, generator=g) * 0.05).cuda()
    b = (torch.randn(N, generator=g) * 0.1).cuda()
    D = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_dense(A, W, b, D, BN=BN, relu=True, split_k=1).set_pair()
    p.run()
    torch.cuda.synchronize()
    ref = (A.float().cpu() @ W.float().cpu().T + b.cpu()).clamp_min(0)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("N,act", [(3072, 2), (2304, 0)])
def test_gemm_auto_pair_wide_n_vs_torch(dev, N, act):
    """ViT/BERT-shaped GEMMs (one wave of 128-row tiles, N >= 2048) take the
    CTA-pair kernel automatically; GELU (exact-form erf) and plain epilogues
    vs a torch fp32 reference."""
    M, K = 148 * 128 + 77, 768
    g = torch.Generator().manual_seed(N + act)
    A = _bf(torch.randn(M, K, generator=g)).cuda()
    W = _bf(torch.randn(N, K, generator=g) * 0.05).cuda()
    b = (torch.randn(N, generator=g) * 0.1).cuda()
    D = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_dense(A, W, b, D, BN=256, act=act)
    assert p.info()["grid_x"] % 2 == 0 and p.info()["stages"] != dev.plan_dense(A, W, b, D, BN=256, act=act,
                                                                                  pair=False).info()["stages"]
    p.run()
    torch.cuda.synchronize()
    ref = A.float() @ W.float().T + b
    if act == 2:
        ref = torch.nn.functional.gelu(ref)
    ok, err, scale = _close(D.float(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin,Cout,k,s,pad,tile,BN", [
    (4, 56, 64, 192, 3, 1, 1, (1, 8, 16), 192), (3, 28, 96, 96, 3, 2, 1, (1, 7, 14), 96),
    (5, 7, 160, 224, 3, 1, 1, (2, 7, 7), 224),
])
def test_conv_cta_pair_vs_torch(dev, n, H, Cin, Cout, k, s, pad, tile, BN):
    g = torch.Generator().manual_seed(n * H + Cin + 1)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, k, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    OH = (H + 2 * pad - k) // s + 1
    D = torch.zeros(n * OH * OH, Cout, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X, n, H, H, Cin, Cin, k, k, s, pad, packed.cuda(), Cout, b.cuda(), D, ldd=Cout,
                      BN=BN, relu=True, tile=tile).set_pair()
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=s, padding=pad).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


def test_coupled_queue_policy_on_device_matches_reference_goldens(dev):
    """ms_policy_apply (the whole OPTIMIZED apply_policy in one launch) on
    the 440 reference-generated EDF queues: every job's final candidate and
    every drop bit-exact; then the fine-grid variant against the host mirror."""
    import numpy as np
    from queue_cases import build_queue, load_cases, outcome
    from paper_2310_18481_b200.policy import DevicePolicy, Policy, apply_policy
    pol = DevicePolicy(max_jobs=4, max_cand=2, ws_bytes=1 << 10)  # tables and scratch grow on demand
    for case in load_cases():
        q, jobs, fb = build_queue(case)
        dropped = pol.apply(q, case["now_us"], fb)
        assert outcome(jobs, dropped) == case["expected"], case["profile"]
    assert pol.launches > 400
    # a 37 us knapsack quantum (the batched server's regime) vs the host mirror
    fine = DevicePolicy(max_jobs=64, max_cand=64, grid_us=37, ws_bytes=512 << 20)
    rng = np.random.default_rng(1)
    for case in [c for i, c in enumerate(load_cases()) if i % 4 == 0]:
        f = float(rng.uniform(0.3, 3.0))
        case = dict(case, factor=f)
        q1, j1, fb1 = build_queue(case)
        q2, j2, fb2 = build_queue(case)
        d1 = fine.apply(q1, case["now_us"], fb1)
        d2 = apply_policy(Policy.OPTIMIZED, q2, case["now_us"], fb2, grid_us=37)
        assert outcome(j1, d1) == outcome(j2, d2)


def test_device_policy_long_queues_without_host_fallback(dev):
    """Queues beyond round 1's 4,096-entry shared table (200 jobs x up to
    9 candidates, TBN serving-regime frontiers, 20 us quantum): device ==
    host mirror, and a queue beyond ms_policy_max_jobs raises instead of
    silently running the host policy."""
    import numpy as np
    from paper_2310_18481_b200.planner import build_matrix, recommended_alphas
    from paper_2310_18481_b200.policy import (DevicePolicy, FeedbackState, Job, JobQueue, Policy, apply_policy,
                                              candidates_with_rounding)
    from paper_2310_18481_b200.profiler import TBN_ACCURACY, PassCostModel, marginal_profile
    enc = [[400 + 55 * n for n in range(96)], [410 + 62 * n for n in range(96)], [420 + 68 * n for n in range(96)]]
    pa = [(1, 577), (4, 881), (8, 1358), (16, 2203), (24, 2848), (32, 3642), (48, 5046), (96, 9183)]
    prof = marginal_profile(PassCostModel(enc, [30.0] * 96, 15, pass_all_us=pa), ("rgb", "flow", "audio"),
                            TBN_ACCURACY, 8)
    mat = build_matrix(prof, range(1, 25), recommended_alphas(prof))
    pol = DevicePolicy(grid_us=20)

    def mk(n_jobs, seed):
        q = JobQueue()
        r2 = np.random.default_rng(seed)
        for i in range(n_jobs):
            size = int(min(24, max(1, round(r2.normal(1, 6)))))
            slo = float(r2.uniform(0.0, 0.6))
            cands = candidates_with_rounding(mat, size, slo)
            if not cands:
                continue
            j = Job(i + 1, 0, size, slo, int(r2.uniform(2_000, 40_000)), cands)
            j.assigned_idx = len(cands) - 1
            q.admit(j)
        return q

    for n_jobs, seed in ((200, 1), (160, 2)):
        q1, q2 = mk(n_jobs, seed), mk(n_jobs, seed)
        d1 = pol.apply(q1, 0, FeedbackState())
        d2 = apply_policy(Policy.OPTIMIZED, q2, 0, FeedbackState(), grid_us=20)
        assert [j.id for j in d1] == [j.id for j in d2]
        assert [j.assigned_idx for j in q1.jobs()] == [j.assigned_idx for j in q2.jobs()]
    assert dev.lib().ms_policy_max_jobs(16) >= 700
    c = candidates_with_rounding(mat, 1, 0.0)
    limit = dev.lib().ms_policy_max_jobs(len(c))
    with pytest.raises(ValueError):
        big = JobQueue()
        for i in range(limit + 1):
            j = Job(i + 1, 0, 1, 0.0, 20_000, c)
            j.assigned_idx = len(c) - 1
            big.admit(j)
        DevicePolicy(grid_us=20).apply(big, 0, FeedbackState())


def test_strategy_dp_on_device_matches_reference_matrices(dev, tmp_path):
    """ms_strategy_dp (offline min-latency table, strategy.py:139-177) builds
    the identical (latency, part-count) table, and the matrices built from it
    are byte-identical to the reference's documents; then a large table
    (S=64, K=4 synthetic) against the host mirror."""
    from pathlib import Path
    import numpy as np
    from paper_2310_18481_b200.planner import (DeviceTable, _Table, build_matrix_device, recommended_alphas,
                                              save_matrix)
    from paper_2310_18481_b200.registry import SynthSpec, load_profile, synth_profile
    golden = Path(__file__).resolve().parent / "golden"
    for path in sorted((golden / "profiles").glob("*.yaml")):
        prof = load_profile(path)
        d, h = DeviceTable(prof, 8), _Table(prof, 8)
        assert np.array_equal(d.lat, h.lat) and np.array_equal(d.cnt, h.cnt), path.stem
        out = tmp_path / f"{path.stem}.json"
        save_matrix(build_matrix_device(prof, range(1, 9), recommended_alphas(prof)), out)
        assert out.read_text() == (golden / "matrices" / f"{path.stem}.json").read_text(), path.stem
    prof = synth_profile(SynthSpec(n_modalities=4, max_batch=8), 3)
    d, h = DeviceTable(prof, 64), _Table(prof, 64)
    assert np.array_equal(d.lat, h.lat) and np.array_equal(d.cnt, h.cnt)


@pytest.mark.parametrize("n,H,Cin,Cout,BN", [(3, 14, 64, 96, 96), (2, 28, 96, 96, 96), (2, 28, 160, 224, 224),
                                             (1, 56, 64, 192, 192), (2, 14, 192, 320, 160), (4, 28, 64, 64, 64)])
def test_conv_halo_vs_torch(dev, n, H, Cin, Cout, BN):
    """3x3/1/1 implicit GEMM with halo reuse (MODE_CONV_HALO): the 9 taps are
    shifted shared-memory views of one (bh+2) x ceil8(W+2) halo box per
    64-channel chunk; output written into a channel slice of a wider tensor."""
    g = torch.Generator().manual_seed(n * H + Cin + 11)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, 3, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    ldd, col0 = Cout + 64, 32
    D = torch.full((n * H * H, ldd), 3.0, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, 1, 1, packed.cuda(), Cout, b.cuda(), D, ldd=ldd, col0=col0,
                      BN=BN, relu=True, halo=True)
    p.run()
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=1, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D[:, col0:col0 + Cout].cpu(), ref)
    assert ok, (err, scale)
    assert torch.all(D[:, :col0] == 3.0) and torch.all(D[:, col0 + Cout:] == 3.0)


@pytest.mark.parametrize("n,H,Cin,Cout,s,tile", [(3, 28, 96, 96, 1, (1, 4, 28)), (2, 28, 96, 96, 2, (1, 8, 14)),
                                                 (2, 14, 160, 224, 1, (1, 7, 14)), (2, 7, 224, 224, 1, (2, 7, 7))])
def test_conv_k32_vs_torch(dev, n, H, Cin, Cout, s, tile):
    """3x3 conv with K over (tap, 32-channel part) halves (MODE_CONV_K32): no
    per-tap channel padding for 96/160/224 input channels."""
    from paper_2310_18481_b200.encoders import pack_conv_weight_k32, pick_bn
    g = torch.Generator().manual_seed(n * H + Cin + 23)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(Cout, Cin, 3, 3, generator=g) * (2.0 / (Cin * 9)) ** 0.5)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    OH = (H + 2 - 3) // s + 1
    D = torch.zeros(n * OH * OH, Cout, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, s, 1, pack_conv_weight_k32(w).cuda(), Cout, b.cuda(), D,
                      ldd=Cout, BN=pick_bn(Cout), relu=True, tile=tile, k32=True)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=s, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D.cpu(), ref)
    assert ok, (err, scale)


def test_fused_compaction_multi_modality_slots_vs_torch(dev):
    """The single-launch ms_compact (index + all modalities' gathers in one
    persistent kernel, units spanning modalities): plain bf16 rows, uint8
    4-channel framed rows and planar 12-channel rows through per-modality
    slot maps, N = 700 mixed masks -- every gathered row equals the torch
    gather, index outputs equal the oracle."""
    import ctypes
    L = dev.lib()
    N, K = 700, 3
    rng = np.random.default_rng(5)
    masks = rng.integers(1, 1 << K, size=N)
    mask = torch.as_tensor(masks.astype(np.int16)).cuda()
    pool0 = _bf(torch.randn(900, 256)).cuda()
    fr, fh, w, pad, pad_h = 2, 5, 48, 3, 3  # 16-B aligned u8 lines (48 x 3, 48 x 10)
    pool1 = torch.randint(0, 256, (800, fr * fh, w, 3), dtype=torch.uint8).cuda()
    pool2 = torch.randint(0, 256, (750, fr * fh, w, 10), dtype=torch.uint8).cuda()
    slot = torch.as_tensor(np.concatenate([rng.permutation(900)[:N], rng.permutation(800)[:N],
                                           rng.permutation(750)[:N]]).astype(np.int32)).cuda()
    G0 = torch.zeros(N, 256, dtype=torch.bfloat16, device="cuda")
    G1 = torch.zeros(N, fr, fh + 2 * pad_h, w + 2 * pad, 4, dtype=torch.bfloat16, device="cuda")
    G2 = torch.zeros(3, N * fr * fh, w + 2 * pad, 4, dtype=torch.bfloat16, device="cuda")
    rows = (dev.RowDesc * 3)(dev.RowDesc(1, 1, 256, 256, 0, 0, 1.0, 0.0, 0, 0, 0),
                             dev.RowDesc(fr * fh, w, 3, 4, pad, 1, 1.0 / 64.0, -2.0, fh, pad_h, N),
                             dev.RowDesc(fr * fh, w, 10, 12, pad, 1, 1.0 / 64.0, -2.0, 0, 0, 2 * N,
                                         N * fr * fh * (w + 2 * pad) * 4))
    X = (ctypes.c_void_p * 3)(pool0.data_ptr(), pool1.data_ptr(), pool2.data_ptr())
    G = (ctypes.c_void_p * 3)(G0.data_ptr(), G1.data_ptr(), G2.data_ptr())
    ix = torch.empty(K * N, dtype=torch.int32, device="cuda")
    inv = torch.empty(K * N, dtype=torch.int32, device="cuda")
    cnt = torch.empty(K, dtype=torch.int32, device="cuda")
    offs = torch.empty((1 << K) + 1, dtype=torch.int32, device="cuda")
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    dev.check(L.ms_compact(mask.data_ptr(), N, K, X, rows, slot.data_ptr(), G, ix.data_ptr(), inv.data_ptr(),
                           cnt.data_ptr(), offs.data_ptr(), perm.data_ptr(), dev.stream_ptr()), "compact")
    torch.cuda.synchronize()
    e_idx, e_inv, e_counts = orc.compact(masks.astype(np.int64), K)
    assert cnt.cpu().tolist() == e_counts.tolist()
    assert np.array_equal(perm.cpu().numpy(), np.argsort(masks, kind="stable"))
    for k in range(K):
        assert np.array_equal(inv.view(K, N)[k].cpu().numpy(), e_inv[k])
    s = slot.long()
    c0, c1, c2 = (int(x) for x in e_counts)
    r0 = s[:N][torch.as_tensor(e_idx[0]).long().cuda()]
    assert torch.equal(G0[:c0], pool0[r0])
    r1 = s[N:2 * N][torch.as_tensor(e_idx[1]).long().cuda()]
    exp1 = (pool1[r1].float() / 64.0 - 2.0).to(torch.bfloat16).view(c1, fr, fh, w, 3)
    assert torch.equal(G1[:c1, :, pad_h:pad_h + fh, pad:pad + w, :3], exp1)
    r2 = s[2 * N:][torch.as_tensor(e_idx[2]).long().cuda()]
    exp2 = (pool2[r2].float() / 64.0 - 2.0).to(torch.bfloat16).view(c2 * fr * fh, w, 10)
    full = torch.zeros(c2 * fr * fh, w, 12, dtype=torch.bfloat16, device="cuda")
    full[..., :10] = exp2
    for q in range(3):
        assert torch.equal(G2[q, :c2 * fr * fh, pad:pad + w], full[..., 4 * q:4 * q + 4])


@pytest.mark.parametrize("n,H,Cin,Cout", [(3, 56, 64, 192), (2, 55, 64, 128), (1, 62, 128, 256), (5, 56, 64, 192),
                                         (3, 64, 64, 192), (2, 64, 128, 128)])
def test_conv_pool_fused_vs_torch_and_unfused(dev, n, H, Cin, Cout):
    """ms_gemm_plan_conv_pool (conv2 + pool2 in one kernel): equal to torch
    fp32 maxpool(relu(conv)) within the bf16 tolerance, and BITWISE equal to
    the unfused halo conv + ms_pool pair (same accumulation order); the
    pooled rows land in a channel slice of a wider tensor, nothing else is
    touched.  H = 55 (odd) and 62 (ceil-mode last window 2 wide); H = 64 is
    the tap-box variant (audio's conv2), compared with the tap-box conv."""
    g = torch.Generator().manual_seed(n * H + Cin + 41)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, 3, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    PH = (H - 3 + 1) // 2 + 1
    ldy, col0 = Cout + 32, 16
    Y = torch.full((n * PH * PH, ldy), 5.0, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv_pool(X, n, H, H, Cin, Cin, packed.cuda(), Cout, b.cuda(), Y, ldy=ldy, col0=col0)
    p.run()
    p.run()
    # unfused: halo conv -> full map, then the 3x3/2 ceil max pool
    D = torch.empty(n * H * H, Cout, dtype=torch.bfloat16, device="cuda")
    if H == 64:  # tap boxes, channel chunk outer like the fused kernel's order when Cin == 64
        from paper_2310_18481_b200.encoders import pick_conv_tile
        q = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, 1, 1, packed.cuda(), Cout, b.cuda(), D, ldd=Cout,
                          BN=Cout, relu=True, tile=pick_conv_tile(n, H, H), pair=False)
    else:
        q = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, 1, 1, packed.cuda(), Cout, b.cuda(), D, ldd=Cout,
                          BN=Cout, relu=True, halo=True)
    q.run()
    Y2 = torch.empty(n * PH * PH, Cout, dtype=torch.bfloat16, device="cuda")
    P = dev.Program()
    P.pool(D, n, H, H, Cout, Cout, 3, 2, 0, True, True, Y2, Cout, 0)
    P.seal()
    P.run()
    torch.cuda.synchronize()
    got = Y[:, col0:col0 + Cout]
    if Cin == 64 or H != 64:  # same accumulation order -> bitwise
        assert torch.equal(got, Y2), (got.float() - Y2.float()).abs().max().item()
    assert torch.all(Y[:, :col0] == 5.0) and torch.all(Y[:, col0 + Cout:] == 5.0)
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=1, padding=1).clamp_min(0)
    ref = torch.nn.functional.max_pool2d(ref, 3, 2, 0, ceil_mode=True)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(got.cpu(), ref)
    assert ok, (err, scale)


@pytest.mark.parametrize("n,H,Cin,Cout", [(3, 28, 96, 96), (2, 14, 128, 128), (1, 56, 64, 192), (3, 28, 64, 96)])
def test_conv_halo_pair_vs_torch(dev, n, H, Cin, Cout):
    """Halo conv on CTA pairs (cta_group::2, M = 256; half of the weights per
    SM, resident when they fit -- the encoders' 28x28 96->96 layers), into a
    channel slice; odd image counts leave the last pair's peer without rows."""
    g = torch.Generator().manual_seed(n * H + Cin + 53)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w, packed = _conv_weights(Cout, Cin, 3, g)
    b = torch.randn(Cout, generator=g) * 0.1
    X = x.permute(0, 2, 3, 1).contiguous().cuda()
    ldd, col0 = Cout + 32, 16
    D = torch.full((n * H * H, ldd), 3.0, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_conv(X, n, H, H, Cin, Cin, 3, 3, 1, 1, packed.cuda(), Cout, b.cuda(), D, ldd=ldd, col0=col0,
                      BN=Cout, relu=True, halo=True).set_pair(True)
    p.run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), w.float(), b, stride=1, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    ok, err, scale = _close(D[:, col0:col0 + Cout].cpu(), ref)
    assert ok, (err, scale)
    assert torch.all(D[:, :col0] == 3.0) and torch.all(D[:, col0 + Cout:] == 3.0)


@pytest.mark.parametrize("N", [1, 37, 256, 1024])
def test_fusion_head_k4_vs_oracle(dev, N):
    """configs[4]'s fusion stage at K = 4 modalities: the device head
    (gather-concat FC1 + ReLU, FC2 -> fp32 logits, split-K with the
    deterministic finalize) over masks covering all 15 subsets, absent
    modalities dropped exactly as the reference drops them (profile.py:157-159:
    zero K blocks), vs the CPU oracle's fusion_forward; rows in request order."""
    from oracle.forward import fusion_forward, fusion_weights as oracle_fusion_weights
    from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead
    K = 4
    g = torch.Generator().manual_seed(400 + N)
    masks = torch.arange(N) % 15 + 1  # every subset, cycled
    masks = masks[torch.randperm(N, generator=g)]
    head = FusionHead(K, 1024, 499, FEAT_DIM)
    full = [_bf(torch.randn(N, FEAT_DIM, generator=g)) for _ in range(K)]
    feats, invs = [], []
    for k in range(K):
        have = ((masks >> k) & 1).bool()
        nk = int(have.sum())
        f = torch.zeros(1024, FEAT_DIM, dtype=torch.bfloat16)
        f[:nk] = full[k][have].to(torch.bfloat16)
        inv = torch.full((N,), -1, dtype=torch.int32)
        inv[have] = torch.arange(nk, dtype=torch.int32)
        feats.append(f.cuda())
        invs.append(inv)
    inv = torch.stack(invs).cuda()
    prog = head.program(N, feats, inv)
    prog.run()
    torch.cuda.synchronize()
    got = head.logits[:N].cpu()
    w = oracle_fusion_weights(K, FEAT_DIM, 499)
    ref = fusion_forward([f.float() for f in full], masks, w)
    ok, err, scale = _close(got, ref)
    assert ok, (err, scale)
    assert (got.argmax(1) == ref.argmax(1)).float().mean().item() >= 0.999
    prog.run()  # deterministic split-K: bitwise identical on a rerun
    torch.cuda.synchronize()
    assert torch.equal(head.logits[:N].cpu(), got)


@pytest.mark.parametrize("n,H,Cin,planes", [(2, 32, 3, 1), (3, 224, 3, 1), (1, 30, 3, 1), (2, 224, 10, 3),
                                            (3, 64, 10, 3)])
def test_stem_fused_1x1_bitwise_vs_stem_then_dense(dev, n, H, Cin, planes):
    """The stem with conv2_red fused (ms_gemm_plan_stem_set_reduce: the pooled
    rows become the A operand of a second MMA in the same kernel) is BITWISE
    equal to the stem writing the pooled map followed by the dense 1x1 GEMM
    (same bf16 pooled values, same K order), for 4-channel and three-plane
    stems, odd pooled widths included."""
    from paper_2310_18481_b200.encoders import (pack_dense_weight, pack_stem_weight, pack_stem_weight_planes,
                                                pack_sw128_weight)
    g = torch.Generator().manual_seed(H + Cin + 29)
    x = _bf(torch.randn(n, Cin, H, H, generator=g))
    w = _bf(torch.randn(64, Cin, 7, 7, generator=g) * (2.0 / (Cin * 49)) ** 0.5)
    b = torch.randn(64, generator=g) * 0.1
    wr = _bf(torch.randn(64, 64, generator=g) * (2.0 / 64) ** 0.5)
    br = torch.randn(64, generator=g) * 0.1
    Hp = H + 6
    if planes == 1:
        X = torch.zeros(n, Hp, Hp, 4, dtype=torch.bfloat16)
        X[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
        Wst, kw = pack_stem_weight(w), {}
    else:
        X = torch.zeros(3, n, Hp, Hp, 4, dtype=torch.bfloat16)
        xp = torch.zeros(n, Hp, Hp, 12, dtype=torch.bfloat16)
        xp[:, 3:H + 3, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
        for q in range(3):
            X[q] = xp[..., 4 * q:4 * q + 4]
        Wst, kw = pack_stem_weight_planes(w), {"planes": 3, "plane_stride": n * Hp * Hp * 4}
    Xd, Wd, bd = X.cuda(), Wst.cuda(), b.cuda()
    OH = (H + 6 - 7) // 2 + 1
    PH = -(-(OH - 3) // 2) + 1
    P1 = torch.empty(n * PH * PH, 64, dtype=torch.bfloat16, device="cuda")
    dev.plan_stem_pool(Xd, n, H, H, 7, 3, Wd, bd, P1, ldy=64, **kw).run()
    R0 = torch.empty(n * PH * PH, 64, dtype=torch.bfloat16, device="cuda")
    dev.plan_dense(P1, pack_dense_weight(wr).cuda(), br.cuda(), R0, M=n * PH * PH, K=64, BN=64, relu=True).run()
    ldr, col0 = 96, 16
    R1 = torch.full((n * PH * PH, ldr), 7.0, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_stem_pool(Xd, n, H, H, 7, 3, Wd, bd, P1, ldy=64, **kw)
    dev.stem_set_reduce(p, pack_sw128_weight(wr).cuda(), br.cuda(), R1[:, col0:], ldy=ldr)
    p.run()
    p.run()
    torch.cuda.synchronize()
    assert torch.equal(R1[:, col0:col0 + 64], R0), (R1[:, col0:col0 + 64].float() - R0.float()).abs().max().item()
    assert torch.all(R1[:, :col0] == 7.0) and torch.all(R1[:, col0 + 64:] == 7.0)


@pytest.mark.parametrize("K,N", [(4, 1), (4, 37), (3, 96), (3, 128), (4, 200), (3, 1024)])
def test_fused_head_cluster_vs_unfused_and_oracle(dev, K, N):
    """The one-launch head (ms_gemm_plan_fused_head: 8-CTA clusters, FC1 and
    FC2 partials reduce-scattered over distributed shared memory) vs the
    unfused three-launch head and the CPU oracle's fusion_forward, all 2^K - 1
    modality subsets, ragged last request tile; bitwise identical on rerun."""
    from oracle.forward import fusion_forward, fusion_weights as oracle_fusion_weights
    from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead
    g = torch.Generator().manual_seed(700 + N + K)
    nsub = (1 << K) - 1
    masks = torch.arange(N) % nsub + 1
    masks = masks[torch.randperm(N, generator=g)]
    head = FusionHead(K, 1024, 499, FEAT_DIM)
    full = [_bf(torch.randn(N, FEAT_DIM, generator=g)) for _ in range(K)]
    feats, invs = [], []
    for k in range(K):
        have = ((masks >> k) & 1).bool()
        nk = int(have.sum())
        f = torch.zeros(1024, FEAT_DIM, dtype=torch.bfloat16)
        f[:nk] = full[k][have].to(torch.bfloat16)
        inv = torch.full((N,), -1, dtype=torch.int32)
        inv[have] = torch.arange(nk, dtype=torch.int32)
        feats.append(f.cuda())
        invs.append(inv)
    inv = torch.stack(invs).cuda()
    prog = head.program(N, feats, inv, fused=False)
    prog.run()
    torch.cuda.synchronize()
    unfused = head.logits[:N].cpu().clone()
    out = torch.full((N + 1, head.n_classes), 7.0, device="cuda")
    p = dev.plan_fused_head(feats, inv, head.w1, head.b1, head.w2, head.b2, out, M=N, feat_dim=FEAT_DIM)
    p.run()
    torch.cuda.synchronize()
    got = out[:N].cpu()
    assert torch.all(out[N] == 7.0)  # no row past M written
    w = oracle_fusion_weights(K, FEAT_DIM, 499)
    ref = fusion_forward([f.float() for f in full], masks, w)
    ok, err, scale = _close(got, ref)
    assert ok, (err, scale)
    ok, err, scale = _close(got, unfused, tol=1e-2)
    assert ok, (err, scale)
    assert (got.argmax(1) == unfused.argmax(1)).float().mean().item() >= 0.99
    p.run()
    torch.cuda.synchronize()
    assert torch.equal(out[:N].cpu(), got)


@pytest.mark.parametrize("K,N", [(4, 1), (3, 5), (4, 16), (3, 33), (4, 70)])
def test_head_gemv_vs_unfused_and_oracle(dev, K, N):
    """The small-pass head (ms_gemm_plan_head_gemv: FC1 weight stream over 128
    CTAs -> bf16 h -> PDL-chained FC2) vs the unfused three-launch head and the
    CPU oracle's fusion_forward over all 2^K - 1 modality subsets; no row past
    M written; bitwise identical on rerun."""
    from oracle.forward import fusion_forward, fusion_weights as oracle_fusion_weights
    from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead
    g = torch.Generator().manual_seed(900 + N + K)
    nsub = (1 << K) - 1
    masks = (torch.arange(N) % nsub + 1)[torch.randperm(N, generator=g)]
    head = FusionHead(K, 1024, 499, FEAT_DIM)
    full = [_bf(torch.randn(N, FEAT_DIM, generator=g)) for _ in range(K)]
    feats, invs = [], []
    for k in range(K):
        have = ((masks >> k) & 1).bool()
        nk = int(have.sum())
        f = torch.zeros(1024, FEAT_DIM, dtype=torch.bfloat16)
        f[:nk] = full[k][have].to(torch.bfloat16)
        inv = torch.full((N,), -1, dtype=torch.int32)
        inv[have] = torch.arange(nk, dtype=torch.int32)
        feats.append(f.cuda())
        invs.append(inv)
    inv = torch.stack(invs).cuda()
    prog = head.program(N, feats, inv, fused=False, gemv=False)
    prog.run()
    torch.cuda.synchronize()
    unfused = head.logits[:N].cpu().clone()
    out = torch.full((N + 1, head.n_classes), 7.0, device="cuda")
    h = torch.empty(N, 512, dtype=torch.bfloat16, device="cuda")
    p = dev.plan_head_gemv(feats, inv, head.w1, head.b1, head.w2, head.b2, out, h, M=N, feat_dim=FEAT_DIM)
    p.run()
    torch.cuda.synchronize()
    got = out[:N].cpu()
    assert torch.all(out[N] == 7.0)
    w = oracle_fusion_weights(K, FEAT_DIM, 499)
    ref = fusion_forward([f.float() for f in full], masks, w)
    ok, err, scale = _close(got, ref)
    assert ok, (err, scale)
    ok, err, scale = _close(got, unfused, tol=1e-2)
    assert ok, (err, scale)
    assert (got.argmax(1) == unfused.argmax(1)).float().mean().item() >= 0.99
    p.run()
    torch.cuda.synchronize()
    assert torch.equal(out[:N].cpu(), got)
    # the served dispatch picks it for small passes
    if N <= head.GEMV_MAX_REQ:
        assert "head_gemv" in head.program(N, feats, inv).ops[0][1].label
