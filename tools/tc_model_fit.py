"""Builder tool: fit the tcgen05 kind::f16 accumulation to a truncating multi-term adder
model (addends aligned to the largest exponent, each truncated toward zero to 23+g bits
below it, exact sum, result truncated to 24 bits) -- which g reproduces the hardware?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_tc_numerics import cases, probe  # noqa: E402


def trunc_to(v, q):  # toward zero to a multiple of q (q a power of two)
    return np.trunc(v / q) * q


def rz24(v):
    out = np.zeros_like(v)
    nz = v != 0
    e = np.floor(np.log2(np.abs(v[nz])))
    q = 2.0 ** (e - 23)
    out[nz] = np.trunc(v[nz] / q) * q
    return out


def model(prev, prods, g, mode):
    add = np.concatenate([prev[..., None], prods], -1)
    mx = np.abs(add).max(-1)
    E = np.floor(np.log2(np.where(mx > 0, mx, 1.0)))
    q = 2.0 ** (E - 23 - g)
    if mode == "rz":
        t = trunc_to(add, q[..., None])
    else:  # floor (two's complement)
        t = np.floor(add / q[..., None]) * q[..., None]
    return rz24(t.sum(-1))


for name, A, B in cases():
    A64, B64, out = probe(A, B)
    ks = out.shape[0]
    res = {}
    for mode in ("rz", "floor"):
        for g in range(0, 7):
            prev = np.zeros((128, 32))
            match = tot = 0
            for s in range(ks):
                a, b = A64[:, 16 * s:16 * s + 16], B64[:, 16 * s:16 * s + 16]
                prods = a[:, None, :] * b[None, :, :]
                m = model(prev, prods, g, mode)
                c = out[s].astype(np.float64)
                match += int((m == c).sum())
                tot += c.size
                prev = c
            res[f"{mode}{g}"] = round(match / tot, 5)
    print(name, res, flush=True)
