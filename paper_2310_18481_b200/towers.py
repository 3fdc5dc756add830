"""configs[2]: VQA-style two-tower model — ViT-B/16 image tower + BERT-base
text tower (random init), masked late fusion, image tower droppable under a
tight SLO (the reference has no model, only the combo
table profile.py:164-174).

Both towers expose the encoder interface ``executor.MaskedModel`` expects
(``x`` input buffer for the compacted sub-batch, ``out`` features
``[max_req, 768]``, ``program(n)``, ``flops(n)``), so compaction, the masked
fusion head, CUDA graphs, the profiler and the serving loop are shared with
the TBN model.  Dense layers are tcgen05 GEMM plans (QKV, out-proj with a
fused residual add, MLP with fused GELU, pooler with fused tanh); LayerNorm,
attention (mma.sync flash-style), patchify and embeddings are
``csrc/transformer.cu``.

Modality bits: 0 = image (ViT), 1 = text (BERT).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import device as dv
from .encoders import pick_bn

D_MODEL, N_HEADS, D_MLP, N_LAYERS = 768, 12, 3072, 12
IMG, PATCH = 224, 16
N_PATCHES = (IMG // PATCH) ** 2          # 196
VIT_TOKENS = N_PATCHES + 1               # 197 with CLS
TEXT_TOKENS, VOCAB, MAX_POS = 40, 30522, 512
VQA_CLASSES = 3129                       # VQA v2 answer vocabulary size


@dataclass(frozen=True)
class TowerSpec:
    name: str
    tokens: int


VQA_MODALITIES = (TowerSpec("image", VIT_TOKENS), TowerSpec("text", TEXT_TOKENS))


def _gen(seed):
    import torch
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    return g


def _lin(g, n_out, n_in, std=0.02):
    import torch
    w = (torch.randn(n_out, n_in, generator=g) * std).to(torch.bfloat16)
    b = (torch.randn(n_out, generator=g) * 0.01).float()
    return w, b


def _ln(g, d):
    import torch
    return (1.0 + 0.05 * torch.randn(d, generator=g)).float(), (0.02 * torch.randn(d, generator=g)).float()


def vit_weights(seed: int):
    """ViT-B/16: patch embedding (K order (kh, kw, c)), CLS, positions,
    12 pre-LN blocks, final LN.  CPU tensors."""
    import torch
    g = _gen(seed)
    W = {"patch": _lin(g, D_MODEL, PATCH * PATCH * 3),
         "cls": (torch.randn(D_MODEL, generator=g) * 0.02).to(torch.bfloat16),
         "pos": (torch.randn(VIT_TOKENS, D_MODEL, generator=g) * 0.02).to(torch.bfloat16)}
    for i in range(N_LAYERS):
        W[f"{i}.ln1"] = _ln(g, D_MODEL)
        W[f"{i}.qkv"] = _lin(g, 3 * D_MODEL, D_MODEL)
        W[f"{i}.proj"] = _lin(g, D_MODEL, D_MODEL)
        W[f"{i}.ln2"] = _ln(g, D_MODEL)
        W[f"{i}.fc1"] = _lin(g, D_MLP, D_MODEL)
        W[f"{i}.fc2"] = _lin(g, D_MODEL, D_MLP)
    W["ln_f"] = _ln(g, D_MODEL)
    return W


def bert_weights(seed: int):
    """BERT-base: word/position/type embeddings + LN, 12 post-LN blocks,
    pooler (dense + tanh on [CLS])."""
    import torch
    g = _gen(seed)
    W = {"word": (torch.randn(VOCAB, D_MODEL, generator=g) * 0.02).to(torch.bfloat16),
         "pos": (torch.randn(MAX_POS, D_MODEL, generator=g) * 0.02).to(torch.bfloat16),
         "type": (torch.randn(2, D_MODEL, generator=g) * 0.02).to(torch.bfloat16),
         "ln_e": _ln(g, D_MODEL)}
    for i in range(N_LAYERS):
        W[f"{i}.qkv"] = _lin(g, 3 * D_MODEL, D_MODEL)
        W[f"{i}.proj"] = _lin(g, D_MODEL, D_MODEL)
        W[f"{i}.ln1"] = _ln(g, D_MODEL)
        W[f"{i}.fc1"] = _lin(g, D_MLP, D_MODEL)
        W[f"{i}.fc2"] = _lin(g, D_MODEL, D_MLP)
        W[f"{i}.ln2"] = _ln(g, D_MODEL)
    W["pooler"] = _lin(g, D_MODEL, D_MODEL)
    return W


def _layer_flops(L):
    return (2 * L * D_MODEL * 3 * D_MODEL + 2 * 2 * L * L * D_MODEL + 2 * L * D_MODEL * D_MODEL
            + 2 * 2 * L * D_MODEL * D_MLP)


def vit_flops_per_image():
    return 2 * N_PATCHES * D_MODEL * PATCH * PATCH * 3 + N_LAYERS * _layer_flops(VIT_TOKENS)


def bert_flops_per_text():
    return N_LAYERS * _layer_flops(TEXT_TOKENS) + 2 * D_MODEL * D_MODEL


class _Tower:
    def _dev_weights(self, W):
        d = self.dev
        self.w = {}
        for k, v in W.items():
            if isinstance(v, tuple):
                self.w[k] = tuple(t.to(d).contiguous() for t in v)
            else:
                self.w[k] = v.to(d).contiguous()

    def program(self, n: int):
        if n not in self._programs:
            if not 1 <= n <= self.max_req:
                raise ValueError(f"n {n} outside 1..{self.max_req}")
            self._programs[n] = self._build(n).seal()
        return self._programs[n]

    def _block_pre_ln(self, P, i, x, h, qkv, a, m, R, L, n):
        """ViT block: x += attn(LN1 x); x += MLP(LN2 x) (residual fused in the GEMMs)."""
        w = self.w
        P.layernorm(x, D_MODEL, R, *w[f"{i}.ln1"], h, D_MODEL, D_MODEL, 1e-6)
        P.gemm(dv.plan_dense(h, w[f"{i}.qkv"][0], w[f"{i}.qkv"][1], qkv, M=R, BN=256))
        P.attention(qkv, 3 * D_MODEL, L, N_HEADS, n, a, D_MODEL, 0.125)
        P.gemm(dv.plan_dense(a, w[f"{i}.proj"][0], w[f"{i}.proj"][1], x, M=R, BN=256, residual=x))
        P.layernorm(x, D_MODEL, R, *w[f"{i}.ln2"], h, D_MODEL, D_MODEL, 1e-6)
        P.gemm(dv.plan_dense(h, w[f"{i}.fc1"][0], w[f"{i}.fc1"][1], m, M=R, BN=256, act=dv.ACT_GELU))
        P.gemm(dv.plan_dense(m, w[f"{i}.fc2"][0], w[f"{i}.fc2"][1], x, M=R, BN=256, residual=x))


class ViTEncoder(_Tower):
    """ViT-B/16 over 224x224 RGB images (compact NHWC bf16) -> CLS feature."""

    def __init__(self, max_req: int, seed: int, device="cuda"):
        import torch
        self.max_req = max_req
        self.dev = torch.device(device)
        self.weights_cpu = vit_weights(seed)
        self._dev_weights(self.weights_cpu)
        bf = torch.bfloat16
        R = max_req * VIT_TOKENS
        self.x = torch.zeros(max_req, IMG, IMG, 3, dtype=bf, device=self.dev)
        self.patches = torch.empty(max_req * N_PATCHES, D_MODEL, dtype=bf, device=self.dev)
        self.pe = torch.empty(max_req * N_PATCHES, D_MODEL, dtype=bf, device=self.dev)
        self.tok = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.h = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.qkv = torch.empty(R, 3 * D_MODEL, dtype=bf, device=self.dev)
        self.a = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.m = torch.empty(R, D_MLP, dtype=bf, device=self.dev)
        self.out = torch.empty(max_req, D_MODEL, dtype=bf, device=self.dev)
        self._programs = {}

    def _build(self, n):
        P = dv.Program()
        w = self.w
        R = n * VIT_TOKENS
        P.patchify(self.x, n, IMG, 3, PATCH, self.patches)
        P.gemm(dv.plan_dense(self.patches, w["patch"][0], w["patch"][1], self.pe, M=n * N_PATCHES,
                             BN=256))
        P.vit_embed(self.pe, w["cls"], w["pos"], n, VIT_TOKENS, D_MODEL, self.tok)
        for i in range(N_LAYERS):
            self._block_pre_ln(P, i, self.tok, self.h, self.qkv, self.a, self.m, R, VIT_TOKENS, n)
        # final LN on the CLS rows only (row stride = one sequence)
        P.layernorm(self.tok, VIT_TOKENS * D_MODEL, n, *w["ln_f"], self.out, D_MODEL, D_MODEL, 1e-6)
        return P

    def flops(self, n: int) -> int:
        return n * vit_flops_per_image()


class BERTEncoder(_Tower):
    """BERT-base over 40-token questions (int32 ids) -> pooled [CLS] feature."""

    def __init__(self, max_req: int, seed: int, device="cuda"):
        import torch
        self.max_req = max_req
        self.dev = torch.device(device)
        self.weights_cpu = bert_weights(seed)
        self._dev_weights(self.weights_cpu)
        bf = torch.bfloat16
        R = max_req * TEXT_TOKENS
        self.x = torch.zeros(max_req, TEXT_TOKENS, dtype=torch.int32, device=self.dev)
        self.tok = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.t = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.qkv = torch.empty(R, 3 * D_MODEL, dtype=bf, device=self.dev)
        self.a = torch.empty(R, D_MODEL, dtype=bf, device=self.dev)
        self.m = torch.empty(R, D_MLP, dtype=bf, device=self.dev)
        self.out = torch.empty(max_req, D_MODEL, dtype=bf, device=self.dev)
        self._programs = {}

    def _build(self, n):
        P = dv.Program()
        w = self.w
        R = n * TEXT_TOKENS
        x, t = self.tok, self.t
        P.bert_embed(self.x, R, TEXT_TOKENS, w["word"], w["pos"], w["type"][0], *w["ln_e"], x, D_MODEL,
                     1e-12)
        for i in range(N_LAYERS):  # post-LN: x = LN(x + attn(x)); x = LN(x + MLP(x))
            P.gemm(dv.plan_dense(x, w[f"{i}.qkv"][0], w[f"{i}.qkv"][1], self.qkv, M=R, BN=256))
            P.attention(self.qkv, 3 * D_MODEL, TEXT_TOKENS, N_HEADS, n, self.a, D_MODEL, 0.125)
            P.gemm(dv.plan_dense(self.a, w[f"{i}.proj"][0], w[f"{i}.proj"][1], t, M=R, BN=256, residual=x))
            P.layernorm(t, D_MODEL, R, *w[f"{i}.ln1"], x, D_MODEL, D_MODEL, 1e-12)
            P.gemm(dv.plan_dense(x, w[f"{i}.fc1"][0], w[f"{i}.fc1"][1], self.m, M=R, BN=256,
                                 act=dv.ACT_GELU))
            P.gemm(dv.plan_dense(self.m, w[f"{i}.fc2"][0], w[f"{i}.fc2"][1], t, M=R, BN=256, residual=x))
            P.layernorm(t, D_MODEL, R, *w[f"{i}.ln2"], x, D_MODEL, D_MODEL, 1e-12)
        # pooler: tanh(W h_cls + b) reading only the CLS rows (row stride 40*768)
        P.gemm(dv.plan_dense(x, w["pooler"][0], w["pooler"][1], self.out, M=n, K=D_MODEL,
                             lda=TEXT_TOKENS * D_MODEL, BN=256, act=dv.ACT_TANH))
        return P

    def flops(self, n: int) -> int:
        return n * bert_flops_per_text()


def build_vqa_model(max_req: int, n_slots: int, seeds=(301, 302), fusion_seed: int = 399,
                    device="cuda", data_seed: int = 0):
    """configs[2]: two-tower model + masked fusion head (1536 -> 512 ->
    3129 answers); image and question pools resident in HBM."""
    import torch
    from .encoders import FusionHead
    from .executor import MaskedModel
    encs = [ViTEncoder(max_req, seeds[0], device), BERTEncoder(max_req, seeds[1], device)]
    head = FusionHead(2, max_req, fusion_seed, D_MODEL, device, n_classes=VQA_CLASSES)
    g = torch.Generator(device=device)
    g.manual_seed(data_seed)
    images = torch.randn((n_slots, IMG, IMG, 3), generator=g, device=device).to(torch.bfloat16)
    ids = torch.randint(0, VOCAB, (n_slots, TEXT_TOKENS), generator=g, device=device, dtype=torch.int32)
    ids[:, 0] = 101  # [CLS]
    # rows in bf16-element units (the gather is byte-exact for int32 ids too)
    rows = [(1, 1, IMG * IMG * 3, IMG * IMG * 3, 0), (1, 1, 2 * TEXT_TOKENS, 2 * TEXT_TOKENS, 0)]
    return MaskedModel(encs, head, [images, ids], rows, max_req, device)
