"""ORACLE — CPU restatement of the forward half of the hot path.

TEST INFRASTRUCTURE ONLY (see oracle/selection.py for the rule).

The reference runs no model: a part's cost is ``profile.part_latency_us``
(sim.py:372-377) and its accuracy a per-combo constant (profile.py:170-174);
the only thing it pins is WHICH modalities a request uses (its assigned
part's mask; dropped set = all_mask & ~mask, profile.py:157-159).  Logits
are therefore "parity unpinned" by the reference.  This module
is the frozen restatement they are checked against:

* plain ``torch.nn.functional`` in fp32 on the CPU, NCHW layout — an
  independent formulation of the same network, not the device's
  implicit-GEMM/NHWC code path;
* the device stores every activation in bf16, so the oracle rounds to bf16
  at exactly those points (conv+ReLU outputs, pool outputs, the segment
  consensus features, the fusion hidden layer) and nowhere else;
* the BN-Inception layer table and every weight generator are restated in
  ``oracle/bninception.py`` independently of the product (Ioffe & Szegedy
  2015 as TSN ships it; the paper's own widths reproduce SURVEY Appendix C's
  MAC counts), so a wrong product layer table or weight order fails parity;
  only the configs[2] towers still take their weights from the product.

Missing-modality rule (builder contract): a request's absent
modality contributes a zero block to the concat, i.e. its FC1 columns are
skipped.  Tolerance (north_star): rtol 2e-2 and >= 99.9 % top-1 agreement.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from oracle import bninception as bni

FEAT_DIM = 1024
N_CLASSES = 97 + 300  # EPIC-100 verbs + nouns
FUSION_HIDDEN = 512


def _bf(x):
    return x.to(torch.bfloat16).float()


def _conv(x, wb, s, p):
    w, b = wb
    return _bf(F.relu(F.conv2d(x, w.float(), b, stride=s, padding=p)))


def bninception_forward(frames, weights, cin: int, size: int, table=bni.TSN):
    """frames: float tensor [n, cin, H, W] (bf16-representable values).
    Returns per-frame feature maps after the last block, fp32 [n, 1024, h, w]
    (not yet pooled or rounded)."""
    x = frames.float()
    for layer in bni.stem(cin):
        if len(layer) == 1:  # 3x3/2 max pool, ceil mode
            x = F.max_pool2d(x, 3, 2, 0, ceil_mode=True)
        else:
            name, _, _, k, s, p = layer
            x = _conv(x, weights[name], s, p)
    for n in bni.ORDER:
        c1, c3r, c3, cdr, cd, pk, proj, s = table[n]
        outs = []
        if c1:
            outs.append(_conv(x, weights[n + "/1x1"], 1, 0))
        t = _conv(x, weights[n + "/3x3_reduce"], 1, 0)
        outs.append(_conv(t, weights[n + "/3x3"], s, 1))
        t = _conv(x, weights[n + "/d3x3_reduce"], 1, 0)
        t = _conv(t, weights[n + "/d3x3_a"], 1, 1)
        outs.append(_conv(t, weights[n + "/d3x3_b"], s, 1))
        if pk == "avg":
            pooled = _bf(F.avg_pool2d(x, 3, 1, 1, count_include_pad=True))
            outs.append(_conv(pooled, weights[n + "/pool_proj"], 1, 0))
        elif pk == "maxproj":
            outs.append(_conv(F.max_pool2d(x, 3, 1, 1), weights[n + "/pool_proj"], 1, 0))
        else:
            outs.append(F.max_pool2d(x, 3, 2, 0, ceil_mode=True))
        x = torch.cat(outs, 1)
    return x


def fusion_weights(n_mod: int, feat_dim: int, seed: int, n_classes: int = N_CLASSES):
    """FC1 (n_mod*feat_dim -> 512, He) + head (512 -> n_classes, LeCun)."""
    (w1, b1), (w2, b2) = bni.dense_weights((n_mod * feat_dim, FUSION_HIDDEN, n_classes), seed, scale_last=1)
    return w1, b1, w2, b2


def encode_requests(clips, weights, cin: int, size: int, segments: int):
    """clips: [n_req, S, H, W, C] NHWC (as stored on the device) ->
    bf16-rounded TSN consensus features [n_req, 1024]."""
    n = clips.shape[0]
    if clips.dtype == torch.uint8:  # uint8 frames/flow: value = u8 / 64 - 2 (exact in bf16)
        clips = clips.float() / 64.0 - 2.0
    frames = clips[..., :cin].float().reshape(n * segments, size, size, cin).permute(0, 3, 1, 2)
    f = bninception_forward(frames, weights, cin, size)  # [n*S, 1024, h, w]
    f = f.reshape(n, segments, f.shape[1], -1).mean(dim=(1, 3))
    return _bf(f)


def mlp_forward(x, layers):
    h = x.float()
    for w, b in layers:
        h = _bf(F.relu(h @ w.float().T + b))
    return h


def fusion_forward(feats, masks, weights):
    """feats: list over modalities of [n_req, F] features for EVERY request
    (rows of absent modalities ignored); masks: int [n_req]."""
    w1, b1, w2, b2 = weights
    n = masks.shape[0]
    cols = []
    for k, f in enumerate(feats):
        present = ((masks >> k) & 1).bool().reshape(n, 1)
        cols.append(torch.where(present, f.float(), torch.zeros_like(f.float())))
    z = torch.cat(cols, 1)
    h = _bf(F.relu(z @ w1.float().T + b1))
    return h @ w2.float().T + b2


class OracleTBN:
    """Whole TBN-shaped model on the CPU: per-modality BN-Inception +
    segment consensus + masked fusion head."""

    def __init__(self, modalities, seeds, fusion_seed: int, segments: int):
        self.mods = modalities
        self.S = segments
        self.enc_w = [bni.weights(m.channels, s) for m, s in zip(modalities, seeds)]
        self.fus_w = fusion_weights(len(modalities), FEAT_DIM, fusion_seed)

    def logits(self, clips_per_mod, masks):
        """clips_per_mod[k]: [n_req, S, H, W, C] for every request (absent
        modalities are not encoded)."""
        n = masks.shape[0]
        feats = []
        for k, m in enumerate(self.mods):
            f = torch.zeros(n, FEAT_DIM)
            sel = torch.nonzero((masks >> k) & 1).flatten()
            if sel.numel():
                f[sel] = encode_requests(clips_per_mod[k][sel], self.enc_w[k], m.channels, m.size,
                                         self.S)
            feats.append(f)
        return fusion_forward(feats, masks, self.fus_w)


class OracleMLP:
    """configs[0]: per-modality MLP towers + masked fusion head."""

    def __init__(self, in_dims, seeds, fusion_seed: int, hidden=(1024, 1024)):
        self.towers = [bni.dense_weights((d,) + tuple(hidden), s) for d, s in zip(in_dims, seeds)]
        self.fus_w = fusion_weights(len(in_dims), hidden[-1], fusion_seed)

    def logits(self, inputs, masks):
        feats = [mlp_forward(x, t) for x, t in zip(inputs, self.towers)]
        return fusion_forward(feats, masks, self.fus_w)


# ---------------------------------------------------------------- configs[2]
# ViT-B/16 + BERT-base two-tower.  Same rules: fp32 math,
# bf16 rounding where the device stores (LN outputs, QKV, attention output,
# the residual stream, MLP hidden, features).


def _lin(x, wb, act=None):
    w, b = wb
    y = x @ w.float().T + b
    if act == "gelu":
        y = F.gelu(y)
    elif act == "tanh":
        y = torch.tanh(y)
    return y


def _ln(x, gb, eps):
    g, b = gb
    return F.layer_norm(x, (x.shape[-1],), g, b, eps)


def _attn(qkv, L, H):
    n = qkv.shape[0] // L
    q, k, v = qkv.reshape(n, L, 3, H, 64).permute(2, 0, 3, 1, 4)
    p = torch.softmax(q @ k.transpose(-1, -2) * 0.125, dim=-1)
    return (p @ v).permute(0, 2, 1, 3).reshape(n * L, H * 64)


def vit_forward(images, W):
    """images [n, 224, 224, 3] NHWC -> CLS features [n, 768] (bf16-rounded)."""
    from paper_2310_18481_b200.towers import N_LAYERS, N_PATCHES, PATCH, VIT_TOKENS
    n = images.shape[0]
    G = images.shape[1] // PATCH
    p = images.float().reshape(n, G, PATCH, G, PATCH, 3).permute(0, 1, 3, 2, 4, 5)
    p = p.reshape(n * N_PATCHES, PATCH * PATCH * 3)
    pe = _bf(_lin(p, W["patch"])).reshape(n, N_PATCHES, -1)
    x = torch.cat([W["cls"].float().expand(n, 1, -1), pe], 1) + W["pos"].float()
    x = _bf(x).reshape(n * VIT_TOKENS, -1)
    for i in range(N_LAYERS):
        h = _bf(_ln(x, W[f"{i}.ln1"], 1e-6))
        a = _bf(_attn(_bf(_lin(h, W[f"{i}.qkv"])), VIT_TOKENS, 12))
        x = _bf(x + _lin(a, W[f"{i}.proj"]))
        h = _bf(_ln(x, W[f"{i}.ln2"], 1e-6))
        m = _bf(_lin(h, W[f"{i}.fc1"], "gelu"))
        x = _bf(x + _lin(m, W[f"{i}.fc2"]))
    cls = x.reshape(n, VIT_TOKENS, -1)[:, 0]
    return _bf(_ln(cls, W["ln_f"], 1e-6))


def bert_forward(ids, W):
    """ids [n, 40] int -> pooled [CLS] features [n, 768] (bf16-rounded)."""
    from paper_2310_18481_b200.towers import N_LAYERS, TEXT_TOKENS
    n = ids.shape[0]
    e = W["word"].float()[ids.long()] + W["pos"].float()[:TEXT_TOKENS] + W["type"].float()[0]
    x = _bf(_ln(e, W["ln_e"], 1e-12)).reshape(n * TEXT_TOKENS, -1)
    for i in range(N_LAYERS):
        a = _bf(_attn(_bf(_lin(x, W[f"{i}.qkv"])), TEXT_TOKENS, 12))
        t = _bf(x + _lin(a, W[f"{i}.proj"]))
        x = _bf(_ln(t, W[f"{i}.ln1"], 1e-12))
        m = _bf(_lin(x, W[f"{i}.fc1"], "gelu"))
        t = _bf(x + _lin(m, W[f"{i}.fc2"]))
        x = _bf(_ln(t, W[f"{i}.ln2"], 1e-12))
    cls = x.reshape(n, TEXT_TOKENS, -1)[:, 0]
    return _bf(_lin(cls, W["pooler"], "tanh"))


class OracleVQA:
    """configs[2] on the CPU: ViT + BERT towers, masked fusion (bit 0 image,
    bit 1 text)."""

    def __init__(self, seeds=(301, 302), fusion_seed: int = 399):
        from paper_2310_18481_b200.towers import VQA_CLASSES, bert_weights, vit_weights
        self.vit_w = vit_weights(seeds[0])
        self.bert_w = bert_weights(seeds[1])
        self.fus_w = fusion_weights(2, 768, fusion_seed, VQA_CLASSES)

    def logits(self, images, ids, masks):
        n = masks.shape[0]
        feats = [torch.zeros(n, 768), torch.zeros(n, 768)]
        sel = torch.nonzero(masks & 1).flatten()
        if sel.numel():
            feats[0][sel] = vit_forward(images[sel], self.vit_w)
        sel = torch.nonzero((masks >> 1) & 1).flatten()
        if sel.numel():
            feats[1][sel] = bert_forward(ids[sel], self.bert_w)
        return fusion_forward(feats, masks, self.fus_w)
