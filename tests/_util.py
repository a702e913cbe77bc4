import numpy as np
import torch

import oracle as O


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def host(t):
    if t.dtype == torch.bfloat16:
        return t.float().cpu().numpy()
    return t.cpu().numpy()


def bf16(a):
    """numpy float32 rounded to bf16 (RNE), still float32 (exactly representable)."""
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def fp8_decode(b, fmt):
    b = np.asarray(b, np.uint8).astype(np.int64)
    s = (b >> 7) & 1
    if fmt == O.E4M3 or fmt == 0:
        e, m = (b >> 3) & 0xF, b & 7
        v = np.where(e == 0, m * 2.0 ** -9, (1 + m / 8.0) * 2.0 ** (e - 7))
    else:
        e, m = (b >> 2) & 0x1F, b & 3
        v = np.where(e == 0, m * 2.0 ** -16, (1 + m / 4.0) * 2.0 ** (e - 15))
    return np.where(s == 1, -v, v).astype(np.float32)


def adversarial(r, c, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((r, c)).astype(np.float32)
    if r > 0:
        x[0] = 0
    if r > 1:
        x[1] = (np.arange(c) % 255 - 127).astype(np.float32)
        x[1, 0] = 127.0
        x[1, 1::4] = 63.5
    if r > 2:
        x[2] *= np.float32(1e-39)
    if r > 3:
        x[3, ::7] *= 100.0
    if r > 4:
        x[4] *= np.float32(3e37)
    if r > 5:
        p = (np.arange(c) % 127) * 2 + 1
        x[5] = (p / 2.0 * 2.0 / 127.0).astype(np.float32)
        x[5, 0] = 2.0
    if r > 6:
        x[6] = rng.integers(-3, 4, c).astype(np.float32) * np.float32(2.0 ** -130)
    return x


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
