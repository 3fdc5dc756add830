"""Host-side layouts of the fused stem (no GPU): the weight packings and the
conv the kernel computes from them, restated on CPU in plain torch.

The kernel's MMAs read B in the no-swizzle core-matrix order (8 n x 8 k
blocks of 128 B, K step 128 B, N step 512 B).  Unpacking that order and
running the kernel's own sum -- over input rows j of a conv-row pair, window
pixels and channels -- must reproduce F.conv2d, which pins the packing and
the row-pair algebra (B_j = [W_j ; W_(j-2)]) without a device."""
import pytest
import torch
import torch.nn.functional as F

from paper_2310_18481_b200.encoders import pack_stem_weight, pack_stem_weight_planes


def _unpack(flat, blocks, n):
    """core-matrix order -> [blocks, n, 32]"""
    return flat.float().reshape(blocks, n // 8, 4, 8, 8).permute(0, 1, 3, 2, 4).reshape(blocks, n, 32)


def _windows(xp, r, ow):
    """the A rows of padded input row r: output pixel ow -> 8 px x 4 ch (32 values) at byte 16*ow"""
    row = xp[r]                                  # [Wp, 4]
    return torch.stack([row[2 * o:2 * o + 8].reshape(32) for o in range(ow)])


@pytest.mark.parametrize("cin", [1, 3])
def test_row_pair_weights_reproduce_conv(cin):
    g = torch.Generator().manual_seed(cin)
    H = 16
    x = torch.randn(cin, H, H, generator=g)
    w = torch.randn(64, cin, 7, 7, generator=g)
    B = _unpack(pack_stem_weight(w), 9, 128)     # [9, 128, 32]
    xp = torch.zeros(H + 6, H + 6, 4)
    xp[3:H + 3, 3:H + 3, :cin] = x.permute(1, 2, 0)
    OH = H // 2
    ref = F.conv2d(x[None].bfloat16().float(), w.bfloat16().float(), stride=2, padding=3)[0]  # [64, OH, OW]
    for r in range(0, OH - 1, 2):               # conv-row pair (r, r+1): input rows 2r + j, j = 0..8
        acc = torch.zeros(OH, 128)
        for j in range(9):
            acc += _windows(xp.bfloat16().float(), 2 * r + j, OH) @ B[j].T
        torch.testing.assert_close(acc[:, :64].T, ref[:, r], rtol=1e-4, atol=1e-3)
        torch.testing.assert_close(acc[:, 64:].T, ref[:, r + 1], rtol=1e-4, atol=1e-3)


def test_plane_weights_reproduce_conv():
    g = torch.Generator().manual_seed(7)
    H, cin = 16, 10
    x = torch.randn(cin, H, H, generator=g)
    w = torch.randn(64, cin, 7, 7, generator=g)
    B = _unpack(pack_stem_weight_planes(w), 21, 64).reshape(7, 3, 64, 32)
    xp = torch.zeros(H + 6, H + 6, 12)
    xp[3:H + 3, 3:H + 3, :cin] = x.permute(1, 2, 0)
    planes = [xp[..., 4 * q:4 * q + 4].bfloat16().float() for q in range(3)]
    OH = H // 2
    ref = F.conv2d(x[None].bfloat16().float(), w.bfloat16().float(), stride=2, padding=3)[0]
    for r in range(OH):
        acc = torch.zeros(OH, 64)
        for kh in range(7):
            for q in range(3):
                acc += _windows(planes[q], 2 * r + kh, OH) @ B[kh, q].T
        torch.testing.assert_close(acc.T, ref[:, r], rtol=1e-4, atol=1e-3)
