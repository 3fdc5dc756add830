"""configs[2] two-tower pieces on the B200 vs plain PyTorch fp32 references,
and the whole masked ViT+BERT forward vs the CPU oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2310_18481_b200 import build, device
    build.build()
    device.lib()
    return device


def _close(got, ref, tol=2e-2):
    err = (got.float().cpu() - ref.float().cpu()).abs().max().item()
    scale = ref.float().abs().max().item() + 1e-6
    return err <= tol * scale, err, scale


@pytest.mark.parametrize("rows,C,ldx", [(197 * 3, 768, 768), (5, 768, 197 * 768), (64, 1024, 1024)])
def test_layernorm(dev, rows, C, ldx):
    L = dev.lib()
    X = torch.randn(rows * (ldx // C) if ldx != C else rows, C).to(torch.bfloat16).cuda()
    X = X.reshape(-1)[: (rows - 1) * ldx + C]
    Xfull = torch.zeros((rows - 1) * ldx + C, dtype=torch.bfloat16, device="cuda")
    Xfull.copy_(X)
    g = torch.randn(C).cuda()
    b = torch.randn(C).cuda()
    Y = torch.empty(rows, C, dtype=torch.bfloat16, device="cuda")
    dev.check(L.ms_layernorm(Xfull.data_ptr(), ldx, rows, g.data_ptr(), b.data_ptr(), Y.data_ptr(), C, C,
                             1e-6, dev.stream_ptr()), "ln")
    torch.cuda.synchronize()
    xs = torch.stack([Xfull[r * ldx: r * ldx + C] for r in range(rows)]).float()
    ref = torch.nn.functional.layer_norm(xs, (C,), g.float(), b.float(), 1e-6)
    assert _close(Y, ref, 1e-2)[0]


@pytest.mark.parametrize("L,n,pad", [(197, 3, 0), (40, 5, 0), (64, 2, 0), (1, 4, 0), (256, 2, 0), (129, 3, 64),
                                     (200, 7, 0)])
def test_attention_vs_torch(dev, L, n, pad):
    """The tcgen05 attention (UMMA for Q K^T and P V, S/O in TMEM): every
    query block / key-chunk boundary, L = 1 .. 256, padded row strides."""
    Lb = dev.lib()
    H = 12
    qkv_full = torch.randn(n * L, 3 * H * 64 + pad).to(torch.bfloat16).cuda()
    qkv = qkv_full[:, : 3 * H * 64]
    out = torch.zeros(n * L, H * 64, dtype=torch.bfloat16, device="cuda")
    dev.check(Lb.ms_attention(qkv.data_ptr(), 3 * H * 64 + pad, L, H, n, out.data_ptr(), H * 64, 0.125,
                              dev.stream_ptr()), "attention")
    torch.cuda.synchronize()
    q, k, v = qkv.float().cpu().reshape(n, L, 3, H, 64).permute(2, 0, 3, 1, 4)
    ref = torch.softmax(q @ k.transpose(-1, -2) * 0.125, -1) @ v
    ref = ref.permute(0, 2, 1, 3).reshape(n * L, H * 64)
    ok, err, scale = _close(out, ref)
    assert ok, (err, scale)


def test_attention_rejects_long_sequences(dev):
    qkv = torch.zeros(300, 3 * 64, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(300, 64, dtype=torch.bfloat16, device="cuda")
    rc = dev.lib().ms_attention(qkv.data_ptr(), 3 * 64, 300, 1, 1, out.data_ptr(), 64, 0.125, dev.stream_ptr())
    assert rc != 0


def test_gemm_gelu_tanh_residual(dev):
    g = torch.Generator().manual_seed(3)
    M, K, N = 300, 768, 3072
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    W = (torch.randn(N, K, generator=g) * 0.03).to(torch.bfloat16).cuda()
    b = torch.randn(N, generator=g).cuda() * 0.1
    D = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    dev.plan_dense(A, W, b, D, BN=256, act=dev.ACT_GELU).run()
    R = torch.randn(M, 768, generator=g).to(torch.bfloat16).cuda()
    D2 = R.clone()
    W2 = (torch.randn(768, N, generator=g) * 0.02).to(torch.bfloat16).cuda()
    dev.plan_dense(D, W2, None, D2, BN=256, residual=D2).run()  # in place: D2 += D @ W2^T
    D3 = torch.zeros(M, 768, dtype=torch.bfloat16, device="cuda")
    dev.plan_dense(A, W2[:, :768].contiguous(), None, D3, BN=256, act=dev.ACT_TANH).run()
    torch.cuda.synchronize()
    ref = torch.nn.functional.gelu(A.float().cpu() @ W.float().cpu().T + b.cpu())
    assert _close(D, ref)[0]
    ref2 = R.float().cpu() + D.float().cpu() @ W2.float().cpu().T
    assert _close(D2, ref2)[0]
    ref3 = torch.tanh(A.float().cpu() @ W2[:, :768].float().cpu().T)
    assert _close(D3, ref3)[0]


def test_vqa_two_tower_vs_oracle():
    from oracle.forward import OracleVQA
    from paper_2310_18481_b200 import build
    build.build()
    from paper_2310_18481_b200.towers import build_vqa_model
    model = build_vqa_model(max_req=4, n_slots=4)
    masks = np.array([3, 2, 1, 3])  # both, text only (image tower dropped), image only, both
    slots = np.array([0, 1, 2, 3])
    logits = model.forward(slots, masks).clone()
    torch.cuda.synchronize()
    orc = OracleVQA()
    ref = orc.logits(model.pools[0][:4].float().cpu(), model.pools[1][:4].cpu(), torch.as_tensor(masks))
    err = (logits.cpu() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-2, err
    assert torch.equal(logits.cpu().argmax(1), ref.argmax(1))
    print(f"VQA two-tower: max rel err {err:.2e}")


def test_vqa_two_tower_vs_oracle_32_requests():
    """configs[2] at a serving-sized pass: 32 requests, image tower dropped
    for a third of them, pool rows shuffled."""
    from oracle.forward import OracleVQA
    from paper_2310_18481_b200 import build
    build.build()
    from paper_2310_18481_b200.towers import build_vqa_model
    model = build_vqa_model(max_req=32, n_slots=40)
    rng = np.random.default_rng(7)
    masks = rng.choice([3, 2, 1], size=32, p=[0.5, 0.35, 0.15])
    slots = rng.permutation(40)[:32]
    logits = model.forward(slots, masks).clone()
    torch.cuda.synchronize()
    orc = OracleVQA()
    sl = torch.as_tensor(slots).long()
    ref = orc.logits(model.pools[0].cpu()[sl].float(), model.pools[1].cpu()[sl], torch.as_tensor(masks))
    scale = ref.abs().max().item()
    err = (logits.cpu() - ref).abs().max().item()
    assert err <= 2e-2 * scale, (err, scale)
    srt = ref.sort(1, descending=True).values
    agree = (logits.cpu().argmax(1) == ref.argmax(1)) | (srt[:, 0] - srt[:, 1] <= 2e-2 * scale)
    assert agree.float().mean().item() >= 0.999
