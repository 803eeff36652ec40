"""Test helper: the band-limited FMM's defining sum, evaluated without any tree
translation. With shared grids every far-field stage is an exact phase shift,
so the multilevel matvec (mlfmm.cpp:361-406) equals, to rounding,

    u_i = sum_{j near i} lambda_j phi(|x_i - x_j|)
        + sum_{j far from i} lambda_j Re sum_m omega C_m e^{i xi_m . (x_i - x_j)}

where "near" is the 3^d leaf neighbourhood of the reference's clamp binning
(geometry.cpp:254-262, 284-293), xi_m the uniform left-endpoint grid
(bandlimit.cpp:269-292), omega = dxi^d and C_m the translation spectrum
(bandlimit.cpp:388-447, lowrank_eval bandlimit.cpp:449). This pins the
restatement in d = 3, where the reference (2-D points only) cannot run: the
identity is checked against the reference itself in d = 2.
"""
import math

import numpy as np


def phi(spec: str, r):
    name, _, par = spec.partition(":")
    c = float(par.split("=")[1]) if par else 1.0
    if name in ("gaussian", "ga"):
        return np.exp(-c * r * r)
    q = np.sqrt(r * r + c * c)
    return 1.0 / q if name == "imq" else q


def lowrank_split_sum(x, w, spec, sigma, m, leaf, c_table):
    """x: [n, d] in [0, 1]^d; c_table: the K = m^d translation spectrum."""
    n, d = x.shape
    nb = 1 << leaf
    idx = np.clip((x * nb).astype(np.int64), 0, nb - 1)
    lid = np.zeros(n, dtype=np.int64)
    for k in range(d):
        lid = lid * nb + idx[:, k]
    dxi = 2.0 * sigma / m
    ax = -sigma + np.arange(m) * dxi
    nodes = np.stack([g.reshape(-1) for g in np.meshgrid(*([ax] * d), indexing="ij")], 1)
    wc = (dxi ** d) * np.asarray(c_table, dtype=np.float64)
    E = np.exp(1j * (x @ nodes.T))  # [n, K]
    u = np.zeros(n)
    for a in np.unique(lid):
        t = np.nonzero(lid == a)[0]
        near = np.all(np.abs(idx - idx[t[0]]) <= 1, axis=1)
        lam_far = np.where(near, 0.0, w)
        far = (E[t] * (wc * (lam_far @ np.conj(E)))[None, :]).sum(1).real
        r = np.sqrt(((x[t, None, :] - x[None, near, :]) ** 2).sum(-1))
        u[t] = far + phi(spec, r) @ w[near]
    return u
