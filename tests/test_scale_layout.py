"""The block-scaled tensor-core scale-factor layout (R15b), stated three ways.

1. `blocked`: index arithmetic -- 512-B tiles of 128 rows x 4 scale columns,
   tiles row-band-major, byte (r % 32) * 16 + ((r // 32) % 4) * 4 + c % 4.
2. `blocked_reshape`: the reshape/permute form cuBLAS documents and torch's
   own reference (`to_blocked`) uses: view (nrb, 128, ncb, 4) -> permute to
   (nrb, ncb, 128, 4) -> (.., 4, 32, 4) -> swap the 4 and 32 axes.
3. `blocked_cute`: CUTLASS's Sm1xx SfKMajorAtom, a CuTe layout of shape
   ((32, 4), (16, 4)) with stride ((16, 4), (0, 1)) in (row, k) coordinates
   (k = element index, 16 elements share a scale), tiled with the K mode
   fastest (tile_to_shape(..., Step<_2, _1>)).
All three must agree, including the zero padding of partial tiles.
"""
import numpy as np
import torch


def blocked(lin: np.ndarray) -> np.ndarray:
    rows, ncol = lin.shape
    nrb, ncb = -(-rows // 128), -(-ncol // 4)
    out = np.zeros(nrb * ncb * 512, np.uint8)
    r, c = np.meshgrid(np.arange(rows), np.arange(ncol), indexing="ij")
    off = ((r // 128) * ncb + c // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + c % 4
    out[off.ravel()] = lin.ravel()
    return out


def blocked_reshape(lin: np.ndarray) -> np.ndarray:
    rows, ncol = lin.shape
    nrb, ncb = -(-rows // 128), -(-ncol // 4)
    pad = torch.zeros(nrb * 128, ncb * 4, dtype=torch.uint8)
    pad[:rows, :ncol] = torch.from_numpy(lin)
    blocks = pad.view(nrb, 128, ncb, 4).permute(0, 2, 1, 3)
    return blocks.reshape(-1, 4, 32, 4).transpose(1, 2).reshape(-1).numpy()


def blocked_cute(lin: np.ndarray) -> np.ndarray:
    rows, ncol = lin.shape
    nrb, ncb = -(-rows // 128), -(-ncol // 4)
    out = np.zeros(nrb * ncb * 512, np.uint8)
    for r in range(rows):
        for j in range(ncol):
            k = 16 * j                                   # first element of scale column j
            m0, m1 = (r % 128) % 32, (r % 128) // 32     # row mode (32, 4), stride (16, 4)
            k0, k1 = k % 16, (k // 16) % 4               # k mode (16, 4), stride (0, 1)
            atom = m0 * 16 + m1 * 4 + k0 * 0 + k1 * 1
            tile = (r // 128) * ncb + (j // 4)           # K-mode tiles fastest
            out[tile * 512 + atom] = lin[r, j]
    return out


def test_three_statements_agree():
    rng = np.random.default_rng(0)
    for rows, ncol in [(1, 1), (37, 6), (128, 4), (129, 5), (257, 64), (300, 13)]:
        lin = rng.integers(1, 127, (rows, ncol), dtype=np.uint8)
        a, b, c = blocked(lin), blocked_reshape(lin), blocked_cute(lin)
        assert np.array_equal(a, b) and np.array_equal(a, c)
        assert a.size == 512 * (-(-rows // 128)) * (-(-ncol // 4))
        assert np.count_nonzero(a) == lin.size            # padding stays zero
