"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libref_lowprec.so).

Run in the dev container (needs /root/reference to build oracle/_ref):
    make -f oracle/Makefile && python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs /root/reference.
Inputs follow the reference's own generators (gaussian_matrix / derive_seed,
matrix.cpp:77-92) plus adversarial rows (zeros, exact half-step ties, outliers,
denormals) from SURVEY.md §8d.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

R = O.ref()


def ref_gauss(r, c, mean, std, seed):
    out = np.empty((r, c), np.float32)
    assert R.ref_gaussian_matrix(r, c, mean, std, seed, out) == 0
    return out


def bf16_round(a):
    """Round float32 to the nearest bf16 (RNE), returned as float32."""
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def adversarial(r, c, seed):
    x = ref_gauss(r, c, 0.0, 1.0, seed)
    x[0] = 0.0                                       # all-zero row -> sentinel 1.0
    if r > 1:
        x[1] = np.arange(c, dtype=np.float32) % 9 - 4  # integer grid
        x[1, 0] = 127.0                               # state 127 -> exact ties 63.5 etc.
        x[1, 1:c:3] = 63.5
    if r > 2:
        x[2] *= 1e-39                                 # denormal row
    if r > 3:
        x[3, ::5] *= 100.0                            # outlier columns
    if r > 4:
        x[4] *= 3.0e37                                # huge magnitudes
    if r > 5:
        # exact half-step ties: p/2 * s / 127 for odd p
        s = 2.0
        p = (np.arange(c) % 127) * 2 + 1
        x[5] = (p / 2.0 * s / 127.0).astype(np.float32)
        x[5, 0] = s
    return x


def quant_case(x):
    out = {}
    r, c = x.shape
    for ax, name in ((0, "row"), (1, "col"), (2, "tensor"), (3, "tensor_t")):
        q = np.empty((c, r) if ax == 3 else (r, c), np.int8)
        st = np.empty(r if ax == 0 else c if ax == 1 else 1, np.float32)
        assert R.ref_quantize_int8(np.ascontiguousarray(x), r, c, ax, q, st) == 0, R.ref_last_error()
        out[f"q_{name}"], out[f"s_{name}"] = q, st
        if ax < 3:
            y = np.empty((r, c), np.float32)
            assert R.ref_dequantize_int8(q, st, ax, r, c, y) == 0
            out[f"deq_{name}"] = y
    for fi, fname in ((0, "e4m3"), (1, "e5m2")):
        for ax, name in ((0, "row"), (1, "col"), (2, "tensor")):
            p = np.empty((r, c), np.float32)
            st = np.empty(r if ax == 0 else c if ax == 1 else 1, np.float32)
            assert R.ref_quantize_fp8(np.ascontiguousarray(x), r, c, fi, ax, p, st) == 0
            out[f"fp8_{fname}_{name}"], out[f"fp8s_{fname}_{name}"] = p, st
    return out


def linear_case(b, n, m, seed, variants=(0, 1, 2, 3, 4), fp8=True):
    x = bf16_round(ref_gauss(b, n, 0.0, 1.0, R.ref_derive_seed(seed, 1)))
    w = bf16_round(ref_gauss(m, n, 0.0, 1.0 / np.sqrt(n), R.ref_derive_seed(seed, 2)))
    g = bf16_round(ref_gauss(b, m, 0.0, 1.0, R.ref_derive_seed(seed, 3)))
    out = {"x": x, "w": w, "g": g}
    for fmt in ((0, 1) if fp8 else (0,)):
        for v in variants:
            y = np.empty((b, m), np.float32)
            dx = np.empty((b, n), np.float32)
            dw = np.empty((m, n), np.float32)
            rc = R.ref_linear_fwd_bwd(v, fmt, x, w, g.ctypes.data, b, n, m, y.ctypes.data, dx.ctypes.data, dw.ctypes.data)
            assert rc == 0, R.ref_last_error()
            out[f"y_{fmt}_{v}"], out[f"dx_{fmt}_{v}"], out[f"dw_{fmt}_{v}"] = y, dx, dw
    return out


def optim_case(seed=7, steps=6):
    shapes = [(4, 6), (3, 3), (17, 33)]
    out = {}
    for clipping in (0, 1, 2):
        thetas = [ref_gauss(r, c, 0.0, 1.0, seed + i).ravel().copy() for i, (r, c) in enumerate(shapes)]
        vs = [np.zeros(r * c, np.float32) for r, c in shapes]
        us = [np.zeros(r * c, np.float32) for r, c in shapes]
        out[f"theta0_{clipping}"] = np.concatenate(thetas)
        rms_all, eta_all, grads_all = [], [], []
        for t in range(1, steps + 1):
            grads = [ref_gauss(r, c, 0.0, 1.0 + (t % 3), 100 * t + i).ravel().copy() for i, (r, c) in enumerate(shapes)]
            grads_all.append(np.concatenate(grads))
            rms, eta = O.stableadamw_step(thetas, grads, vs, us, t, alpha=0.01, weight_decay=0.1, clipping=clipping,
                                          max_grad_norm=1.0, use_ref=True)
            rms_all.append(rms)
            eta_all.append(eta)
        out[f"grads_{clipping}"] = np.stack(grads_all)
        out[f"theta_{clipping}"] = np.concatenate(thetas)
        out[f"v_{clipping}"] = np.concatenate(vs)
        out[f"u_{clipping}"] = np.concatenate(us)
        out[f"rms_{clipping}"] = np.stack(rms_all)
        out[f"eta_{clipping}"] = np.stack(eta_all)
    out["shapes"] = np.array(shapes, np.int64)
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), **quant_case(adversarial(13, 70, 11)),
                        **{f"g_{k}": v for k, v in quant_case(ref_gauss(37, 53, 0.0, 1.5, 42)).items()},
                        x_adv=adversarial(13, 70, 11), x_g=ref_gauss(37, 53, 0.0, 1.5, 42))
    np.savez_compressed(os.path.join(HERE, "linear_small.npz"), **linear_case(37, 53, 29, 5))
    np.savez_compressed(os.path.join(HERE, "linear_aligned.npz"), **linear_case(160, 128, 96, 42, variants=(0, 1, 2, 3, 4)))
    np.savez_compressed(os.path.join(HERE, "optimizer.npz"), **optim_case())
    vals = {}
    for fi, name in ((0, "e4m3"), (1, "e5m2")):
        v = np.empty(256, np.float32)
        k = R.ref_fp8_value_set(fi, v)
        vals[name] = v[:k]
    np.savez_compressed(os.path.join(HERE, "fp8_value_sets.npz"), **vals)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
