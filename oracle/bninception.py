"""ORACLE — BN-Inception layer table and weights, written independently of
the product (``paper_2310_18481_b200/encoders.py``).

TEST INFRASTRUCTURE ONLY (see oracle/selection.py for the rule).

The table is Ioffe & Szegedy 2015 (arXiv 1502.03167), Figure 5 ("Inception
architecture" with batch normalisation), as the TSN/TBN Caffe model ships it
(``bn_inception.prototxt``: inception_4c/1x1 has 128 outputs and
inception_4d/1x1 has 64, so every 4x block emits 576 channels; the paper's
figure lists 160 and 96).  ``IOFFE`` is the figure as printed; SURVEY
Appendix C's analytic MAC counts (2.032 / 2.307 / 2.551 GMAC per frame at
3x224^2 / 10x224^2 / 1x256^2) are reproduced from it in
tests/test_oracle.py, and ``TSN`` differs from it in exactly those two
widths.  BatchNorm is folded into each conv's bias (inference).

Columns: (#1x1, #3x3 reduce, #3x3, double #3x3 reduce, double #3x3,
pool, pool projection, stride).  pool: "avg" 3x3/1 average + 1x1
projection, "max" 3x3/2 max pass-through (stride-2 blocks), "maxproj"
3x3/1 max + 1x1 projection (5b).
"""

from __future__ import annotations

IOFFE = {
    "3a": (64, 64, 64, 64, 96, "avg", 32, 1),
    "3b": (64, 64, 96, 64, 96, "avg", 64, 1),
    "3c": (0, 128, 160, 64, 96, "max", 0, 2),
    "4a": (224, 64, 96, 96, 128, "avg", 128, 1),
    "4b": (192, 96, 128, 96, 128, "avg", 128, 1),
    "4c": (160, 128, 160, 128, 160, "avg", 128, 1),
    "4d": (96, 128, 192, 160, 192, "avg", 128, 1),
    "4e": (0, 128, 192, 192, 256, "max", 0, 2),
    "5a": (352, 192, 320, 160, 224, "avg", 128, 1),
    "5b": (352, 192, 320, 192, 224, "maxproj", 128, 1),
}
TSN = dict(IOFFE)
TSN["4c"] = (128,) + IOFFE["4c"][1:]
TSN["4d"] = (64,) + IOFFE["4d"][1:]
ORDER = ("3a", "3b", "3c", "4a", "4b", "4c", "4d", "4e", "5a", "5b")


def _out(h, k, s, p, ceil=False):
    span = h + 2 * p - k
    o = (-(-span // s) if ceil else span // s) + 1
    if ceil and (o - 1) * s >= h + p:  # Caffe/PyTorch: the last window must start inside
        o -= 1
    return o


def stem(cin):
    """conv1 7x7/2 p3 -> max 3x3/2 (ceil) -> conv2_red 1x1 -> conv2 3x3 p1 -> max 3x3/2 (ceil)."""
    return [("conv1", cin, 64, 7, 2, 3), ("pool1",), ("conv2_red", 64, 64, 1, 1, 0),
            ("conv2", 64, 192, 3, 1, 1), ("pool2",)]


def convs(cin, table=TSN):
    """Every convolution in weight-generation order: (name, cin, cout, k)."""
    out = [(n, ci, co, k) for n, ci, co, k, *_ in (s for s in stem(cin) if len(s) > 1)]
    c = 192
    for b in ORDER:
        c1, c3r, c3, cdr, cd, pk, proj, _ = table[b]
        if c1:
            out.append((f"{b}/1x1", c, c1, 1))
        out += [(f"{b}/3x3_reduce", c, c3r, 1), (f"{b}/3x3", c3r, c3, 3), (f"{b}/d3x3_reduce", c, cdr, 1),
                (f"{b}/d3x3_a", cdr, cd, 3), (f"{b}/d3x3_b", cd, cd, 3)]
        if proj:
            out.append((f"{b}/pool_proj", c, proj, 1))
        c = c1 + c3 + cd + (proj if proj else c)
    return out


def macs(cin, size, table=TSN):
    """Multiply-accumulates of one frame (real channels)."""
    h = _out(size, 7, 2, 3)
    total = h * h * 64 * cin * 49
    h = _out(h, 3, 2, 0, True)
    total += h * h * 64 * 64 + h * h * 64 * 9 * 192
    h = _out(h, 3, 2, 0, True)
    c = 192
    for b in ORDER:
        c1, c3r, c3, cdr, cd, pk, proj, s = table[b]
        o = _out(h, 3, s, 1)
        total += h * h * c * (c1 + c3r + cdr + proj)
        total += o * o * c3r * 9 * c3 + h * h * cdr * 9 * cd + o * o * cd * 9 * cd
        c = c1 + c3 + cd + (proj if proj else c)
        h = o
    return total


def weights(cin, seed, table=TSN):
    """He-normal conv weights rounded to bf16 and N(0, 0.02) fp32 biases,
    drawn in layer order from one seeded CPU generator: per conv
    randn(cout, cin, k, k) * sqrt(2 / (cin k k)), then randn(cout) * 0.02."""
    import torch
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    W = {}
    for name, ci, co, k in convs(cin, table):
        w = (torch.randn(co, ci, k, k, generator=g) * (2.0 / (ci * k * k)) ** 0.5).to(torch.bfloat16)
        b = (torch.randn(co, generator=g) * 0.02).float()
        W[name] = (w, b)
    return W


def dense_weights(dims, seed, scale_last=None):
    """Linear layers (out, in) drawn in order: randn(out, in) * sqrt(2/in)
    (or sqrt(1/in) for the last when ``scale_last`` == 1) -> bf16, then
    randn(out) * 0.02 biases."""
    import torch
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    out = []
    for i, (din, dout) in enumerate(zip(dims, dims[1:])):
        gain = 1.0 if (scale_last == 1 and i == len(dims) - 2) else 2.0
        w = (torch.randn(dout, din, generator=g) * (gain / din) ** 0.5).to(torch.bfloat16)
        b = (torch.randn(dout, generator=g) * 0.02).float()
        out.append((w, b))
    return out
