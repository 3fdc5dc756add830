"""Per-modality encoders and the late-fusion head, as native op programs.

The reference has no model at all: a part's cost is a table lookup
(sim.py:372-377, profile.py:164-168) and its accuracy a per-combo constant
(profile.py:170-174).  These are the random-init encoders the north_star
names; their numerics are pinned by the frozen
CPU restatement in ``oracle/forward.py`` ("parity unpinned" by the
reference).

* ``TBN_BNINCEPTION``: TSN/TBN-style BN-Inception (69 convolutions, 1024-d
  output; BatchNorm folded into conv bias as at inference) applied to S=3
  segments per request, global-average pooled and averaged over segments
  (TSN consensus).  Inputs per modality: rgb 3x224x224, flow 10x224x224
  (5 stacked x/y frames), audio 1x256x256 spectrogram.
* ``MLP``: configs[0]'s small per-modality MLP towers (D -> 1024 -> 1024).
* ``FusionHead``: masked concat over the present modalities (absent slots
  are zero, i.e. their K columns are skipped) -> FC 3072->512 -> ReLU ->
  verb/noun heads 97+300 = 397 logits.

Every layer maps to one tcgen05 GEMM plan (``csrc/gemm.cu``), a pooling,
im2col or segment-mean op (``csrc/ops.cu``); the list for one (modality,
batch) is sealed into a ``device.Program`` and executed by one native call
(``ms_program_run``), optionally captured in a CUDA graph.

Weights are generated on the CPU from ``torch.manual_seed``-style
generators so the oracle rebuilds them bit-identically.
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

FEAT_DIM = 1024
N_VERBS, N_NOUNS = 97, 300
N_CLASSES = N_VERBS + N_NOUNS
FUSION_HIDDEN = 512
SEGMENTS = 3
CONV1_PAD = 3  # conv1 is 7x7/2 pad 3; its input is stored W-padded by this much

# name, 1x1, 3x3 reduce, 3x3, double-3x3 reduce, double-3x3, pool kind, pool proj, stride
# (TSN's Caffe BN-Inception: 4c 1x1=128, 4d 1x1=64 so every 4x block emits 576)
INCEPTION_BLOCKS = (
    ("3a", 64, 64, 64, 64, 96, "avg", 32, 1),
    ("3b", 64, 64, 96, 64, 96, "avg", 64, 1),
    ("3c", 0, 128, 160, 64, 96, "max", 0, 2),
    ("4a", 224, 64, 96, 96, 128, "avg", 128, 1),
    ("4b", 192, 96, 128, 96, 128, "avg", 128, 1),
    ("4c", 128, 128, 160, 128, 160, "avg", 128, 1),
    ("4d", 64, 128, 192, 160, 192, "avg", 128, 1),
    ("4e", 0, 128, 192, 192, 256, "max", 0, 2),
    ("5a", 352, 192, 320, 160, 224, "avg", 128, 1),
    ("5b", 352, 192, 320, 192, 224, "maxproj", 128, 1),
)


U8_SCALE, U8_BIAS = 1.0 / 64.0, -2.0  # uint8 inputs -> bf16 value u8 * scale + bias (exact)


@dataclass(frozen=True)
class ModalitySpec:
    name: str
    channels: int
    size: int  # square input H = W
    uint8: bool = False  # stored as uint8 in the pools (frames, quantised flow)

    @property
    def cpad(self) -> int:
        """Stored channels of the first conv's input: 4 for <= 4 real channels
        (8-byte pixels: MODE_CONV_C4, one 128-B K block per filter-row pair),
        12 for 5-12 (MODE_CONV_C12), else a multiple of 8 (MODE_CONV_SMALLC)."""
        if self.channels <= 4:
            return 4
        if self.channels <= 12:
            return 12  # 24-byte pixels: MODE_CONV_C12 (three 32-element parts per filter row)
        return -(-self.channels // 8) * 8

    @property
    def row_pad(self) -> int:
        """Zero rows above/below each frame in the first conv's input
        (MODE_CONV_C4/C12 pad rows themselves instead of TMA out-of-bounds fill)."""
        return CONV1_PAD if self.cpad in (4, 12) else 0

    def frame_elems(self) -> int:
        return self.size * self.size * self.cpad


TBN_MODALITIES = (ModalitySpec("rgb", 3, 224, True), ModalitySpec("flow", 10, 224, True),
                  ModalitySpec("audio", 1, 256))


def conv_out(h: int, k: int, s: int, p: int) -> int:
    return (h + 2 * p - k) // s + 1


def pool_out(h: int, k: int, s: int, p: int, ceil_mode: bool) -> int:
    span = h + 2 * p - k
    o = (-(-span // s) if ceil_mode else span // s) + 1
    if ceil_mode and (o - 1) * s >= h + p:
        o -= 1
    return o


def bninception_layers(cin: int, size: int):
    """Static layer list: dicts with kind/name/geometry, in execution order.

    Each conv dict has cin, cout, k, s, p, h (input side) and its MACs per
    frame; pools carry k, s, p, ceil, is_max.  Used by the device builder,
    the oracle and the FLOP count.
    """
    L = []
    h = size
    L.append(dict(kind="conv", name="conv1", cin=cin, cout=64, k=7, s=2, p=3, h=h))
    h = conv_out(h, 7, 2, 3)
    L.append(dict(kind="pool", name="pool1", c=64, k=3, s=2, p=0, ceil=True, is_max=True, h=h))
    h = pool_out(h, 3, 2, 0, True)
    L.append(dict(kind="conv", name="conv2_red", cin=64, cout=64, k=1, s=1, p=0, h=h))
    L.append(dict(kind="conv", name="conv2", cin=64, cout=192, k=3, s=1, p=1, h=h))
    L.append(dict(kind="pool", name="pool2", c=192, k=3, s=2, p=0, ceil=True, is_max=True, h=h))
    h = pool_out(h, 3, 2, 0, True)
    c = 192
    for name, c1, c3r, c3, cdr, cd, pk, proj, s in INCEPTION_BLOCKS:
        out_c = c1 + c3 + cd + (proj if proj else c)
        L.append(dict(kind="block", name=name, cin=c, c1=c1, c3r=c3r, c3=c3, cdr=cdr, cd=cd,
                      pool=pk, proj=proj, s=s, h=h, cout=out_c))
        h = conv_out(h, 3, s, 1) if s == 2 else h
        c = out_c
    L.append(dict(kind="final", c=c, h=h))
    return L


def bninception_macs(cin: int, size: int) -> int:
    """Multiply-accumulates of one frame (real channels, no padding)."""
    total = 0
    for L in bninception_layers(cin, size):
        if L["kind"] == "conv":
            o = conv_out(L["h"], L["k"], L["s"], L["p"])
            total += o * o * L["cout"] * L["cin"] * L["k"] * L["k"]
        elif L["kind"] == "block":
            h, c, s = L["h"], L["cin"], L["s"]
            o = conv_out(h, 3, s, 1) if s == 2 else h
            total += h * h * c * (L["c1"] + L["c3r"] + L["cdr"])  # 1x1s at input size
            total += o * o * L["c3r"] * 9 * L["c3"]
            total += h * h * L["cdr"] * 9 * L["cd"]
            total += o * o * L["cd"] * 9 * L["cd"]
            if L["proj"]:
                total += h * h * c * L["proj"]
    return total


def request_flops(modality: ModalitySpec, segments: int = SEGMENTS) -> int:
    return 2 * segments * bninception_macs(modality.channels, modality.size)


# ------------------------------------------------------------------ weights


def _gen(seed: int):
    import torch
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    return g


def make_conv(g, cout: int, cin: int, k: int):
    """He-normal conv weight (bf16-rounded) + small bias, CPU tensors.
    Weight layout [cout, cin, k, k] (PyTorch), bias fp32."""
    import torch
    w = (torch.randn(cout, cin, k, k, generator=g) * (2.0 / (cin * k * k)) ** 0.5).to(torch.bfloat16)
    b = (torch.randn(cout, generator=g) * 0.02).float()
    return w, b


def bninception_weights(cin: int, size: int, seed: int):
    """Deterministic weights for one modality's encoder: dict name -> (w, b)."""
    g = _gen(seed)
    W = {}
    for L in bninception_layers(cin, size):
        if L["kind"] == "conv":
            W[L["name"]] = make_conv(g, L["cout"], L["cin"], L["k"])
        elif L["kind"] == "block":
            n, c = L["name"], L["cin"]
            if L["c1"]:
                W[n + "/1x1"] = make_conv(g, L["c1"], c, 1)
            W[n + "/3x3_reduce"] = make_conv(g, L["c3r"], c, 1)
            W[n + "/3x3"] = make_conv(g, L["c3"], L["c3r"], 3)
            W[n + "/d3x3_reduce"] = make_conv(g, L["cdr"], c, 1)
            W[n + "/d3x3_a"] = make_conv(g, L["cd"], L["cdr"], 3)
            W[n + "/d3x3_b"] = make_conv(g, L["cd"], L["cd"], 3)
            if L["proj"]:
                W[n + "/pool_proj"] = make_conv(g, L["proj"], c, 1)
    return W


def fusion_weights(n_mod: int, feat_dim: int, seed: int, n_classes: int = N_CLASSES):
    import torch
    g = _gen(seed)
    k = n_mod * feat_dim
    w1 = (torch.randn(FUSION_HIDDEN, k, generator=g) * (2.0 / k) ** 0.5).to(torch.bfloat16)
    b1 = (torch.randn(FUSION_HIDDEN, generator=g) * 0.02).float()
    w2 = (torch.randn(n_classes, FUSION_HIDDEN, generator=g) * (1.0 / FUSION_HIDDEN) ** 0.5).to(torch.bfloat16)
    b2 = (torch.randn(n_classes, generator=g) * 0.02).float()
    return w1, b1, w2, b2


def mlp_weights(dims, seed: int):
    import torch
    g = _gen(seed)
    out = []
    for din, dout in zip(dims, dims[1:]):
        w = (torch.randn(dout, din, generator=g) * (2.0 / din) ** 0.5).to(torch.bfloat16)
        b = (torch.randn(dout, generator=g) * 0.02).float()
        out.append((w, b))
    return out


def pack_conv_weight(w):
    """[cout, cin, k, k] -> [cout, k*k*ceil64(cin)] tap-major, channel-padded
    (the implicit-GEMM K order of ``ms_gemm_plan_conv``)."""
    import torch
    cout, cin, k, _ = w.shape
    cc = -(-cin // 64) * 64
    out = torch.zeros(cout, k * k, cc, dtype=torch.bfloat16)
    out[:, :, :cin] = w.permute(0, 2, 3, 1).reshape(cout, k * k, cin)
    return out.reshape(cout, k * k * cc).contiguous()


def pack_conv_weight_k32(w):
    """[cout, cin, k, k] -> [cout, ceil64(k*k*cin)] in (tap, channel) order
    with no per-tap channel padding (MODE_CONV_K32's K order)."""
    import torch
    cout, cin, k, _ = w.shape
    kk = k * k * cin
    out = torch.zeros(cout, -(-kk // 64) * 64, dtype=torch.bfloat16)
    out[:, :kk] = w.permute(0, 2, 3, 1).reshape(cout, kk)
    return out.contiguous()


def pack_smallc_weight(w, cpad: int):
    """[cout, cin, kh, kw] -> [cout, kh * 8 * cpad]: K ordered (kh, window
    pixel j < 8, channel) with channels zero-padded to ``cpad`` and taps
    j >= kw zero (MODE_CONV_SMALLC's K order)."""
    import torch
    cout, cin, kh, kw = w.shape
    wp = torch.zeros(cout, kh, 8, cpad, dtype=torch.bfloat16)
    wp[:, :, :kw, :cin] = w.permute(0, 2, 3, 1)
    return wp.reshape(cout, kh * 8 * cpad).contiguous()


def pack_c4_weight(w):
    """[cout, cin <= 4, kh <= 8, kw <= 8] -> [cout, ceil(kh/2) * 64]: K block
    kb holds filter rows (2kb, 2kb+1), each as 8 window pixels x 4 channels
    (MODE_CONV_C4's K order; missing rows/taps/channels are zero)."""
    import torch
    cout, cin, kh, kw = w.shape
    nkb = -(-kh // 2)
    wp = torch.zeros(cout, nkb * 2, 8, 4, dtype=torch.bfloat16)
    wp[:, :kh, :kw, :cin] = w.permute(0, 2, 3, 1)
    return wp.reshape(cout, nkb * 64).contiguous()


def pack_stem_weight(w):
    """[64, cin <= 4, 7, 7] -> the fused stem's row-pair weights (MODE_STEM_POOL):
    for each of the 9 input rows j of a conv-row pair (r, r+1), B_j = [W_j ;
    W_(j-2)] (128 x 32: output channels of row r, then of row r+1; W_kh =
    filter row kh as 8 window pixels x 4 channels, zero outside 0..6), stored
    in the no-swizzle UMMA core-matrix order (8 n x 8 k blocks of 128 B; K
    step 128 B, N step 512 B), 9 x 8 KB."""
    import torch
    cout, cin, kh, kw = w.shape
    assert cout == 64 and kh == 7 and kw <= 8 and cin <= 4
    wk = torch.zeros(9, 64, 8, 4, dtype=torch.float32)       # filter rows, padded to 9 (7, 8 zero)
    wk[:kh, :, :kw, :cin] = w.float().permute(2, 0, 3, 1)
    wk = wk.reshape(9, 64, 32)
    b = torch.zeros(9, 128, 32, dtype=torch.float32)
    b[:, :64] = wk                                            # row r: W_j
    b[2:, 64:] = wk[:7]                                       # row r+1: W_(j-2)
    b = b.reshape(9, 16, 8, 4, 8).permute(0, 1, 3, 2, 4)     # (j, n/8, k/8, n%8, k%8)
    return b.reshape(-1).to(torch.bfloat16).contiguous()


def pack_stem_weight_planes(w, planes: int = 3):
    """[64, cin <= 4*planes, 7, 7] -> the planar fused stem's weights: per
    (filter row kh, 4-channel plane) a 64 x 32 block (8 window pixels x 4
    channels of that plane), no-swizzle core-matrix order (K step 128 B, N step
    512 B), blocks in (kh, plane) order."""
    import torch
    cout, cin, kh, kw = w.shape
    assert cout == 64 and kh == 7 and kw <= 8 and cin <= 4 * planes
    wk = torch.zeros(kh, 64, 8, 4 * planes, dtype=torch.float32)
    wk[:, :, :kw, :cin] = w.float().permute(2, 0, 3, 1)
    wk = wk.reshape(kh, 64, 8, planes, 4).permute(0, 3, 1, 2, 4).reshape(kh, planes, 64, 32)
    b = wk.reshape(kh, planes, 8, 8, 4, 8).permute(0, 1, 2, 4, 3, 5)  # (kh, pl, n/8, k/8, n%8, k%8)
    return b.reshape(-1).to(torch.bfloat16).contiguous()


def pack_c12_weight(w):
    """[cout, cin <= 12, kh <= 8, kw <= 8] -> [cout, ceil(3*kh/2) * 64]: K =
    (filter row, 8 window pixels x 12 channels = 96) rows back to back, zero
    padded to whole 64-element blocks (MODE_CONV_C12's K order)."""
    import torch
    cout, cin, kh, kw = w.shape
    nkb = -(-3 * kh // 2)
    wp = torch.zeros(cout, kh, 8, 12, dtype=torch.bfloat16)
    wp[:, :, :kw, :cin] = w.permute(0, 2, 3, 1)
    out = torch.zeros(cout, nkb * 64, dtype=torch.bfloat16)
    out[:, : kh * 96] = wp.reshape(cout, kh * 96)
    return out.contiguous()


def pack_im2col_weight(w, k_pad: int):
    """[cout, cin, k, k] -> [cout, k_pad] in im2col order (kh, kw, c)."""
    import torch
    cout, cin, k, _ = w.shape
    out = torch.zeros(cout, k_pad, dtype=torch.bfloat16)
    out[:, : k * k * cin] = w.permute(0, 2, 3, 1).reshape(cout, k * k * cin)
    return out.contiguous()


def pack_dense_weight(w):
    """[n, k] -> [n, ceil64(k)] zero padded."""
    import torch
    n, k = w.shape
    kp = -(-k // 64) * 64
    out = torch.zeros(n, kp, dtype=torch.bfloat16)
    out[:, :k] = w
    return out.contiguous()


def pack_sw128_weight(w):
    """[N, 64] bf16 K-major -> the same bytes in the UMMA SW128 K-major layout
    (16-B chunk j of row n at chunk j ^ (n & 7)), so one linear bulk copy puts
    the weights in shared memory ready as a B operand (the stem's fused 1x1)."""
    import torch
    w = w.reshape(w.shape[0], -1).to(torch.bfloat16)
    assert w.shape[1] == 64, "one 128-B swizzle row per output channel"
    n = w.shape[0]
    chunks = w.reshape(n, 8, 8)
    out = torch.empty_like(chunks)
    for r in range(n):
        out[r, [(j ^ (r & 7)) for j in range(8)]] = chunks[r]
    return out.reshape(n, 64).contiguous()


def pick_bn(n: int, m_tiles: int | None = None, target_ctas: int = 96) -> int:
    """Tile width for N output columns: one tile when N <= 256, else the
    fewest equal-ish tiles (multiples of 32).  With ``m_tiles`` given and too
    few (m, n) tiles to occupy ``target_ctas`` SMs, split N further (tiles
    >= 64 wide): each CTA's serial K loop shrinks and idle SMs take the rest.
    (Not used by the TBN encoders: with modality streams and branch lanes
    already sharing the SMs it measured slower, tools/pass_ab.py.)"""
    tiles = -(-n // 256)
    if m_tiles is not None:
        while m_tiles * tiles < target_ctas and -(-n // (tiles + 1)) >= 64:
            tiles += 1
    bn = -(-n // tiles)
    return -(-bn // 32) * 32


def pick_conv_tile(n_img: int, oh: int, ow: int):
    """(bn, bh, bw) with bn*bh*bw <= 128 minimising the number of 128-row
    tiles (ties: larger bw for contiguous TMA rows)."""
    best = None
    for bw in range(1, min(ow, 128) + 1):
        for bh in range(1, min(oh, 128 // bw) + 1):
            per = bh * bw
            for bn in sorted({1, max(1, min(n_img, 128 // per))}):
                if bn * per > 128:
                    continue
                tiles = -(-n_img // bn) * -(-oh // bh) * -(-ow // bw)
                key = (tiles, -bw, -bh)
                if best is None or key < best[0]:
                    best = (key, (bn, bh, bw))
    return best[1]


def conv_m_tiles(n_img: int, o: int, tile) -> int:
    bn, bh, bw = tile
    return -(-n_img // bn) * -(-o // bh) * -(-o // bw)


# ------------------------------------------------------------ device build


class BNInceptionEncoder:
    """One modality's BN-Inception on the device for up to ``max_req``
    requests of ``segments`` frames each.

    ``program(n_req)`` returns a sealed native op program that maps the
    gathered input ``X [n_req*S, H, W, C]`` (NHWC bf16) to features
    ``out [n_req, 1024]`` (bf16).  Buffers are allocated once at capacity;
    programs are cached per request count.
    """

    def __init__(self, modality: ModalitySpec, max_req: int, seed: int, segments: int = SEGMENTS,
                 device="cuda"):
        import torch
        self.mod = modality
        self.max_req = max_req
        self.S = segments
        self.dev = torch.device(device)
        self.layers = bninception_layers(modality.channels, modality.size)
        self.weights_cpu = bninception_weights(modality.channels, modality.size, seed)
        # conv1 + pool1 as one kernel (MS_NO_FUSED_STEM=1: the conv + pool pair, for A/B)
        self.fused_stem = os.environ.get("MS_NO_FUSED_STEM") is None
        # conv2 + pool2 as one kernel (MS_NO_FUSED_POOL2=1: the conv + pool pair, for A/B)
        self.fused_pool2 = os.environ.get("MS_NO_FUSED_POOL2") is None
        # conv2_red fused into the stem (overlapping-row stems, output width <= 112;
        # MS_NO_STEM_RED=1: the separate 1x1 GEMM, for A/B)
        self.stem_red_env = os.environ.get("MS_NO_STEM_RED") is None
        self._pack()
        self._alloc()
        self._programs = {}
        self._lanes = None  # side streams for the Inception branch lanes

    # -- weights on device
    def _pack(self):
        import torch
        d = self.dev
        W = self.weights_cpu
        self.w = {}
        self.b = {}
        for name, (w, b) in W.items():
            if name == "conv1":
                cp = self.mod.cpad
                packer = {4: pack_c4_weight, 12: pack_c12_weight}.get(cp)
                self.w[name] = (packer(w) if packer else pack_smallc_weight(w, cp)).to(d)
                if cp == 4:
                    self.w["stem"] = pack_stem_weight(w).to(d)
                elif cp == 12:
                    self.w["stem"] = pack_stem_weight_planes(w).to(d)
            elif w.shape[-1] == 1:
                self.w[name] = pack_dense_weight(w.reshape(w.shape[0], -1)).to(d)
                if name == "conv2_red":
                    self.w["conv2_red_sw"] = pack_sw128_weight(w.reshape(w.shape[0], -1)).to(d)
            elif w.shape[1] % 64 and w.shape[1] % 32 == 0:
                # 96/160/224 input channels: K = 9*C without per-tap padding
                # (MODE_CONV_K32, 1.04-1.14x, profiles/r01_k32_bench.txt)
                self.w[name] = pack_conv_weight_k32(w).to(d)
            else:
                self.w[name] = pack_conv_weight(w).to(d)
            self.b[name] = b.to(d)
        # merged 1x1 weights/biases per block (1x1 | 3x3_reduce | d3x3_reduce)
        for L in self.layers:
            if L["kind"] != "block":
                continue
            n = L["name"]
            parts = ([n + "/1x1"] if L["c1"] else []) + [n + "/3x3_reduce", n + "/d3x3_reduce"]
            biases = [self.b[p] for p in parts]
            if L["pool"] == "avg":
                # proj(avgpool(x)) == avgpool(proj(x)) for count-include-pad
                # averaging: project at the narrow width inside the merged GEMM
                # (bias and ReLU are applied after the pool)
                parts.append(n + "/pool_proj")
                biases.append(torch.zeros_like(self.b[n + "/pool_proj"]))
            self.w[n + "/merged"] = torch.cat([self.w[p] for p in parts], 0).contiguous()
            self.b[n + "/merged"] = torch.cat(biases, 0).contiguous()

    def _w64(self, name):
        """3x3 weights with each tap's channels padded to 64 (the halo layout),
        for layers whose default packing is MODE_CONV_K32's."""
        if not hasattr(self, "_w64_cache"):
            self._w64_cache = {}
        if name not in self._w64_cache:
            w, _ = self.weights_cpu[name]
            self._w64_cache[name] = pack_conv_weight(w).to(self.dev)
        return self._w64_cache[name]

    # -- activation buffers at capacity
    def _alloc(self):
        import torch
        d = self.dev
        n_img = self.max_req * self.S
        bf = torch.bfloat16

        def buf(pixels, ch):
            return torch.empty(max(1, pixels), ch, dtype=bf, device=d)

        size = self.mod.size
        h1 = conv_out(size, 7, 2, 3)
        self.a_c1 = buf(n_img * h1 * h1, 64)
        h2 = pool_out(h1, 3, 2, 0, True)
        self.a_p1 = buf(n_img * h2 * h2, 64)
        self.a_c2r = buf(n_img * h2 * h2, 64)
        # the unpooled conv2 map exists only without the fused conv2 + pool2 kernel
        self.a_c2 = None if (self.fused_pool2 and (55 <= h2 <= 62 or h2 == 64)) else buf(n_img * h2 * h2, 192)
        self.blocks = {}
        # ping-pong block outputs + scratch sized for the largest block
        max_pix_c = 0
        max_tmp = 0
        for L in self.layers:
            if L["kind"] == "block":
                h, s = L["h"], L["s"]
                o = conv_out(h, 3, s, 1) if s == 2 else h
                max_pix_c = max(max_pix_c, o * o * L["cout"], h * h * L["cin"])
                max_tmp = max(max_tmp, h * h * max(L["c3r"], L["cdr"], L["cd"], L["cin"]))
        self.ping = torch.empty(n_img * max_pix_c, dtype=bf, device=d)
        self.pong = torch.empty(n_img * max_pix_c, dtype=bf, device=d)
        self.t3 = torch.empty(n_img * max_tmp, dtype=bf, device=d)
        self.td = torch.empty(n_img * max_tmp, dtype=bf, device=d)
        self.td2 = torch.empty(n_img * max_tmp, dtype=bf, device=d)
        self.tp = torch.empty(n_img * max_tmp, dtype=bf, device=d)
        self.outs = [torch.empty(self.max_req, FEAT_DIM, dtype=bf, device=d) for _ in range(2)]
        self.out = self.outs[0]
        # conv1 input: W-padded by CONV1_PAD zero pixels per side (the gather
        # pads) and, for 4-channel frames, row-padded too (zero rows written
        # once here, never touched by the gather)
        rp = self.mod.row_pad
        self.x = torch.zeros(n_img, size + 2 * rp, size + 2 * CONV1_PAD, self.mod.cpad, dtype=bf, device=d)
        # fused stem: 4-channel frames as they are; 12-channel (flow) frames as
        # three 4-channel planes in the same buffer (ms_compact writes them)
        h1 = conv_out(size, 7, 2, 3)
        cp = self.mod.cpad
        self.stem_planes = 0
        if self.fused_stem and cp == 4 and h1 <= 128:
            self.stem_planes = 1
        elif self.fused_stem and cp == 12 and h1 <= 112:
            self.stem_planes = 3
        self.x_plane_stride = n_img * (size + 2 * rp) * (size + 2 * CONV1_PAD) * 4 if self.stem_planes == 3 else 0
        # for the 4-channel (rgb) stem the fused 1x1 is slower timed alone
        # (117.6 us vs 74.3 + 27.0) but equal on the served path, where the
        # separate GEMM's HBM round trip competes with the other encoders
        # (tools/ringab.sh, profiles/r02_ringab_stemred.txt); MS_STEM_RED_RGB=0
        # keeps it separate
        self.stem_red = (bool(self.stem_planes) and self.stem_red_env and h1 <= 112
                         and (self.stem_planes == 3 or os.environ.get("MS_STEM_RED_RGB", "1") == "1"))

    # features of pass parity p land in outs[p]: with passes pipelined the next
    # pass's encoder may finish before the previous pass's fusion head has read
    # its features (executor.MaskedModel.run_ring)
    supports_parity = True

    # shared=True: plans for a pass where other encoders run beside this one
    # (two-CTAs-per-SM GEMMs take the second slot only with >= 4 tiles per
    # SM, leaving it to the partners; ms_set_occ2_grid); same buffers
    supports_shared = True
    SHARED_OCC2_GRID = int(os.environ.get("MS_SHARED_OCC2_GRID", "2"))

    def program(self, n_req: int, parity: int = 0, shared: bool = False):
        key = (n_req, parity, bool(shared))
        if key in self._programs:
            return self._programs[key]
        if not 1 <= n_req <= self.max_req:
            raise ValueError(f"n_req {n_req} outside 1..{self.max_req}")
        from . import device as dv
        prev = dv.set_occ2_grid(self.SHARED_OCC2_GRID) if shared else None
        try:
            prog = self._build(n_req, parity)
        finally:
            if shared:
                dv.set_occ2_grid(prev)
        self._programs[key] = prog
        return prog

    def _build(self, n_req: int, parity: int = 0):
        """Trunk (stem, each block's merged 1x1, final pool) plus, per
        Inception block, three concurrent lanes: the double-3x3 chain, the
        3x3 branch and the pool branch (``device.StagedProgram``)."""
        from . import device as dv
        if self._lanes is None:
            self._lanes = dv.LaneContext(2)
        SP = dv.StagedProgram(self._lanes)
        P = dv.Program()
        n = n_req * self.S
        size = self.mod.size
        h1 = conv_out(size, 7, 2, 3)
        # stem: the few-channel 7x7/2 conv reads the frames directly with TMA
        # (channels padded to 8 in memory; no im2col round trip)
        cp = self.mod.cpad
        h2 = pool_out(h1, 3, 2, 0, True)
        # stage 0 = the ops that read the gathered input self.x (the stem): the
        # executor can release self.x to the next pass's compaction after it
        if self.stem_planes:
            # conv1 + bias + ReLU + pool1 in one kernel that feeds the raw padded
            # input rows to the tensor cores (csrc/gemm.cu MODE_STEM_POOL; flow
            # as three 4-channel planes); the unpooled map never reaches HBM
            P.gemm(dv.plan_stem_pool(self.x, n, size, size, 7, 3, self.w["stem"], self.b["conv1"], self.a_p1,
                                     ldy=64, planes=self.stem_planes, plane_stride=self.x_plane_stride))
        else:
            P.gemm(dv.plan_conv(self.x, n, size, size, cp, cp, 7, 7, 2, 3, self.w["conv1"], 64,
                                self.b["conv1"], self.a_c1, ldd=64, BN=64, relu=True,
                                tile=pick_conv_tile(n, h1, h1)))
        SP.stage(P)
        P = dv.Program()
        if not self.stem_planes:
            P.pool(self.a_c1, n, h1, h1, 64, 64, 3, 2, 0, True, True, self.a_p1, 64, 0)
        if self.stem_red:
            # conv2_red (1x1 64->64) fused into the stem: the pooled rows are the
            # A operand of a second MMA in the stem kernel (pool1's map never stored)
            dv.stem_set_reduce(SP.stages[0][0].ops[0][1], self.w["conv2_red_sw"], self.b["conv2_red"],
                               self.a_c2r, ldy=64)
            SP.stages[0][0].ops[0][1].flops += 2 * n * h2 * h2 * 64 * 64
        else:
            P.gemm(dv.plan_dense(self.a_p1, self.w["conv2_red"], self.b["conv2_red"], self.a_c2r,
                                 M=n * h2 * h2, K=64, BN=64, relu=True))
        # conv2 (56x56 rgb/flow): halo reuse measured 1.08-1.09x faster than the
        # tap-box 2-SM kernel (tools/halo_bench.py); narrower layers lose more to
        # the ceil8(W+2)-wide tiles than they gain, audio's 64+2 does not tile 128
        h = pool_out(h2, 3, 2, 0, True)
        cur = self.ping
        if self.fused_pool2 and (55 <= h2 <= 62 or h2 == 64):
            # conv2 + ReLU + pool2 in one kernel (csrc/convpool.cu; halo tiles at 56^2,
            # tap boxes at audio's 64^2): the unpooled x 192 map never reaches HBM;
            # bitwise equal to the pair below (rgb 56^2 at 183 frames: 1.43x)
            P.gemm(dv.plan_conv_pool(self.a_c2r, n, h2, h2, 64, 64, self.w["conv2"], 192, self.b["conv2"],
                                     cur, ldy=192))
        else:
            P.gemm(dv.plan_conv(self.a_c2r, n, h2, h2, 64, 64, 3, 3, 1, 1, self.w["conv2"], 192,
                                self.b["conv2"], self.a_c2, ldd=192, BN=192, relu=True,
                                tile=pick_conv_tile(n, h2, h2), halo=42 <= h2 <= 62))
            P.pool(self.a_c2, n, h2, h2, 192, 192, 3, 2, 0, True, True, cur, 192, 0)
        c = 192
        nxt = self.pong
        for L in self.layers:
            if L["kind"] != "block":
                continue
            lanes = self._block(P, L, n, h, c, cur, nxt)
            SP.stage(P)
            SP.stage(*lanes)
            P = dv.Program()
            h = conv_out(h, 3, L["s"], 1) if L["s"] == 2 else h
            c = L["cout"]
            cur, nxt = nxt, cur
        P.segment_mean(cur, n_req, self.S, h * h, c, self.outs[parity], FEAT_DIM)
        SP.stage(P)
        return SP.seal()

    def _block(self, P, L, n, h, cin, X, Y):
        """Append the block's merged 1x1 GEMM to the trunk ``P``; return its
        independent branch lanes (longest first: it stays on the trunk stream)."""
        from . import device as dv
        name, s = L["name"], L["s"]
        c1, c3r, c3, cdr, cd, proj = L["c1"], L["c3r"], L["c3"], L["cdr"], L["cd"], L["proj"]
        o = conv_out(h, 3, s, 1) if s == 2 else h
        cout = L["cout"]
        pix_in, pix_out = n * h * h, n * o * o
        Xv = X[: pix_in * cin].view(pix_in, cin)
        Yv = Y[: pix_out * cout].view(pix_out, cout)
        T3 = self.t3[: pix_in * c3r].view(pix_in, c3r)
        Td = self.td[: pix_in * cdr].view(pix_in, cdr)
        Td2 = self.td2[: pix_in * cd].view(pix_in, cd)
        # merged 1x1s: [1x1 -> Y slice 0 | 3x3_reduce -> T3 | d3x3_reduce -> Td]
        segs = []
        col = 0
        if c1:
            segs.append((0, c1, Yv, cout, 0))
            col = c1
        segs.append((col, col + c3r, T3, c3r, 0))
        segs.append((col + c3r, col + c3r + cdr, Td, cdr, 0))
        nm = col + c3r + cdr
        fold_pool = L["pool"] == "avg"
        if fold_pool:
            Tq = self.tp[: pix_in * proj].view(pix_in, proj)
            segs.append((nm, nm + proj, Tq, proj, 0, dv.SEG_NO_RELU))
            nm += proj
        # (narrower N tiles that would let the wide merged GEMMs run two CTAs per
        # SM measured slower: 128-wide +3.8 %, <= 224-wide +2 % pass time)
        P.gemm(dv.plan_dense(Xv, self.w[name + "/merged"], self.b[name + "/merged"], Yv, M=pix_in,
                             K=cin, BN=pick_bn(nm), relu=True, segs=segs))
        tile_in = pick_conv_tile(n, h, h)
        tile_out = pick_conv_tile(n, o, o)

        def halo_ok(cin_, cout_, stride_):
            # halo + resident weights (one N tile, 9 x 64-ch blocks in smem): 1.36x the
            # one-CTA-per-SM tap-box kernel at 28x28 alone, but with tap-box plans
            # launched two CTAs per SM (OCC=2) the served pass is 2.2 % faster
            # without it (profiles/r02_ab_halo28.txt): opt-in (MS_HALO28=1)
            pitch = -(-(h + 2) // 8) * 8  # halo row width: must tile the 128-row M block
            return (stride_ == 1 and 14 < h <= 30 and 128 % pitch == 0 and cin_ <= 64 and cout_ <= 128
                    and os.environ.get("MS_HALO28") is not None)

        no_k32 = os.environ.get("MS_NO_K32") is not None  # A/B: 64-padded tap-box instead of K32

        def k32(cin_):  # matches the weight packing in _pack
            return cin_ % 64 != 0 and cin_ % 32 == 0 and not no_k32

        def conv3(X_, cin_, cout_, stride_, wname, D_, ldd_, col0_, tile_):
            """3x3 conv plan: halo (+ CTA pair) where measured faster, else tap-box / K32."""
            if halo_ok(cin_, cout_, stride_):
                return dv.plan_conv(X_, n, h, h, cin_, cin_, 3, 3, 1, 1, self.w[wname], cout_, self.b[wname], D_,
                                    ldd=ldd_, col0=col0_, BN=pick_bn(cout_), relu=True, halo=True)
            if halo_pair_ok(cin_, stride_):
                p_ = dv.plan_conv(X_, n, h, h, cin_, cin_, 3, 3, 1, 1, self._w64(wname), cout_, self.b[wname], D_,
                                  ldd=ldd_, col0=col0_, BN=pick_bn(cout_), relu=True, halo=True)
                return p_.set_pair(True)
            wt = self._w64(wname) if (no_k32 and cin_ % 64) else self.w[wname]
            # (two N tiles for the under-filled 7x7 layers measured +1.4 % pass time)
            return dv.plan_conv(X_, n, h, h, cin_, cin_, 3, 3, stride_, 1, wt, cout_, self.b[wname], D_,
                                ldd=ldd_, col0=col0_, BN=pick_bn(cout_), relu=True, tile=tile_, k32=k32(cin_))

        def halo_pair_ok(cin_, stride_):
            """Halo tiles on CTA pairs with half of the (64-padded) weights
            resident per SM: at 28x28 96->96 1.26x the one-CTA-per-SM K32
            kernel (profiles/r02_conv_variants.txt), but slower than the K32
            kernel two CTAs per SM in the served pass (opt-in: MS_HALO28_PAIR);
            at 14x14 the tap-box kernels win for every served shape
            (MS_HALO14_PAIR)."""
            if stride_ != 1 or 128 % (-(-(h + 2) // 8) * 8) != 0:
                return False
            if 14 < h <= 30:
                return cin_ == 96 and os.environ.get("MS_HALO28_PAIR") is not None
            if h == 14:
                return os.environ.get("MS_HALO14_PAIR") is not None
            return False
        # 3x3 branch (stride s) -> Y[:, c1 : c1+c3]
        B3 = dv.Program()
        B3.gemm(conv3(T3, c3r, c3, s, name + "/3x3", Yv, cout, c1, tile_out))
        # double 3x3: stride 1 then stride s -> Y[:, c1+c3 : c1+c3+cd]
        BD = dv.Program()
        BD.gemm(conv3(Td, cdr, cd, 1, name + "/d3x3_a", Td2, cd, 0, tile_in))
        BD.gemm(conv3(Td2, cd, cd, s, name + "/d3x3_b", Yv, cout, c1 + c3, tile_out))
        pc = c1 + c3 + cd
        BP = dv.Program()
        if fold_pool:  # avgpool of the projected (pre-bias) branch + bias + ReLU
            BP.pool(Tq, n, h, h, proj, proj, 3, 1, 1, False, False, Yv, cout, pc,
                    bias=self.b[name + "/pool_proj"], relu=True)
        elif proj:  # max pool does not commute with the projection
            Tp = self.tp[: pix_in * cin].view(pix_in, cin)
            BP.pool(Xv, n, h, h, cin, cin, 3, 1, 1, False, True, Tp, cin, 0)
            BP.gemm(dv.plan_dense(Tp, self.w[name + "/pool_proj"], self.b[name + "/pool_proj"], Yv,
                                  M=pix_in, K=cin, BN=pick_bn(proj), relu=True, col0=pc, ldd=cout))
        else:  # stride-2 max-pool pass-through into the concat
            BP.pool(Xv, n, h, h, cin, cin, 3, 2, 0, True, True, Yv, cout, pc)
        return [BD, B3, BP]

    def flops(self, n_req: int) -> int:
        return n_req * request_flops(self.mod, self.S)


class MLPEncoder:
    """configs[0]'s per-modality MLP tower D -> 1024 -> 1024 (ReLU)."""

    def __init__(self, in_dim: int, max_req: int, seed: int, hidden=(1024, 1024), device="cuda"):
        import torch
        self.dims = (in_dim,) + tuple(hidden)
        self.max_req = max_req
        self.dev = torch.device(device)
        self.weights_cpu = mlp_weights(self.dims, seed)
        self.w = [pack_dense_weight(w).to(self.dev) for w, _ in self.weights_cpu]
        self.b = [b.to(self.dev) for _, b in self.weights_cpu]
        self.x = torch.empty(max_req, -(-in_dim // 64) * 64, dtype=torch.bfloat16, device=self.dev)
        self.x.zero_()
        self.acts = [torch.empty(max_req, d, dtype=torch.bfloat16, device=self.dev) for d in hidden]
        self.out = self.acts[-1]
        self._programs = {}

    def program(self, n_req: int):
        from . import device as dv
        if n_req in self._programs:
            return self._programs[n_req]
        P = dv.Program()
        src, k = self.x, self.dims[0]
        for (w, b, dst) in zip(self.w, self.b, self.acts):
            P.gemm(dv.plan_dense(src, w, b, dst, M=n_req, K=k, BN=pick_bn(dst.shape[1]), relu=True))
            src, k = dst, dst.shape[1]
        self._programs[n_req] = P.seal()
        return self._programs[n_req]

    def flops(self, n_req: int) -> int:
        return n_req * sum(2 * a * b for a, b in zip(self.dims, self.dims[1:]))


class FusionHead:
    """Masked concat -> FC(K*F -> 512) -> ReLU -> FC(512 -> 397) logits."""

    def __init__(self, n_mod: int, max_req: int, seed: int, feat_dim: int = FEAT_DIM, device="cuda",
                 n_classes: int = N_CLASSES):
        import torch
        self.n_mod = n_mod
        self.feat_dim = feat_dim
        self.max_req = max_req
        self.n_classes = n_classes
        self.dev = torch.device(device)
        self.weights_cpu = fusion_weights(n_mod, feat_dim, seed, n_classes)
        w1, b1, w2, b2 = self.weights_cpu
        self.w1, self.b1 = w1.to(self.dev).contiguous(), b1.to(self.dev)
        self.w2, self.b2 = pack_dense_weight(w2).to(self.dev), b2.to(self.dev)
        self.h = torch.empty(max_req, FUSION_HIDDEN, dtype=torch.bfloat16, device=self.dev)
        self.logits = torch.empty(max_req, n_classes, dtype=torch.float32, device=self.dev)
        self._programs = {}

    # the one-launch head wins up to ~48 requests per 128-request tile
    # (tools/head_time.py, profiles/r02_head_time.txt: 10.9 vs 13.6 us at 1
    # request, K = 3); above that its DSMEM reduce-scatter (~20 B/clk per SM)
    # costs more than the split-K round trip through L2
    FUSED_MAX_REQ = int(os.environ.get("MS_FUSED_HEAD_MAX", "48"))

    @property
    def fusable(self) -> bool:
        """The one-launch cluster head applies (K % 512, classes <= 512);
        MS_FUSED_HEAD=0 keeps the three-launch path (A/B switch)."""
        return (os.environ.get("MS_FUSED_HEAD", "1") != "0" and self.n_classes <= FUSION_HIDDEN
                and (self.n_mod * self.feat_dim) % 512 == 0 and self.feat_dim % 64 == 0)

    # the one-launch weight-streaming head (ms_gemm_plan_head_gemv) below
    # GEMV_MAX_REQ requests: the head is then a 4 MB W1 stream that the
    # cluster head reads with 8 SMs and the GEMV kernel with 128
    GEMV_MAX_REQ = int(os.environ.get("MS_HEAD_GEMV_MAX", "16"))

    @property
    def gemv_ok(self) -> bool:
        return self.feat_dim % 8 == 0 and self.n_mod * self.feat_dim <= 4096

    def program(self, n_req: int, feats, inv, fused=None, gemv=None):
        """feats: per-modality compacted feature buffers; inv [n_mod, >=n_req].
        gemv: None = the weight-streaming GEMV head up to GEMV_MAX_REQ requests
        (when fused is not forced); fused: None = the one-launch cluster head
        when it applies and n_req <= FUSED_MAX_REQ, else the gather GEMM + FC2
        split-K path."""
        from . import device as dv
        if gemv is None:
            gemv = fused is None and self.gemv_ok and n_req <= self.GEMV_MAX_REQ
        fused = (self.fusable and n_req <= self.FUSED_MAX_REQ) if fused is None else fused
        key = (n_req, tuple(f.data_ptr() for f in feats), inv.data_ptr(), fused, gemv)
        if key in self._programs:
            return self._programs[key]
        P = dv.Program()
        if gemv:
            P.gemm(dv.plan_head_gemv(list(feats), inv, self.w1, self.b1, self.w2, self.b2, self.logits, self.h,
                                     M=n_req, feat_dim=self.feat_dim))
            self._programs[key] = P.seal()
            return self._programs[key]
        if fused:
            P.gemm(dv.plan_fused_head(list(feats), inv, self.w1, self.b1, self.w2, self.b2, self.logits, M=n_req,
                                      feat_dim=self.feat_dim))
            self._programs[key] = P.seal()
            return self._programs[key]
        P.gemm(dv.plan_gather(list(feats), inv, self.w1, self.b1, self.h, M=n_req,
                              feat_dim=self.feat_dim, BN=256, relu=True))
        # the fp32 logits leave through the split-K finalize (coalesced rows)
        # instead of the per-thread fp32 epilogue; K parts fill idle SMs
        bn2 = pick_bn(self.n_classes)
        tiles = -(-n_req // 128) * -(-self.n_classes // bn2)
        P.gemm(dv.plan_dense(self.h, self.w2, self.b2, self.logits, M=n_req, K=FUSION_HIDDEN, BN=bn2,
                             out_fp32=True, split_k=max(2, min(FUSION_HIDDEN // 64, 148 // tiles))))
        self._programs[key] = P.seal()
        return self._programs[key]

    def flops(self, n_req: int) -> int:
        return n_req * (2 * self.n_mod * self.feat_dim * FUSION_HIDDEN + 2 * FUSION_HIDDEN * self.n_classes)
