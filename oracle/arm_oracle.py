"""CPU oracle for the 7-DOF sphere-arm collision factor (SURVEY.md §8-f3,
configuration C3) — TEST INFRASTRUCTURE ONLY (PARITY UNPINNED).

The reference (`gvplan`) has no manipulator model: its factor kernel
(`_kernels.pyx:93-129`, contract `_kernels_py.py:16-53`) evaluates the hinge
cost of ONE point, the state's position coordinates. The C3 configuration of
SURVEY.md §8d asks for the same expectation with the robot's body swept by
spheres: psi(q) = sigma * sum_s max(r_s + eps - d(FK_s(q)), 0)^2, q the 7 joint
angles (the first half of the 14-dimensional state), d the trilinear SDF of the
reference (sdf.py:80-122). This module restates that definition directly — a
standard-DH forward kinematics, every sigma point, sequential accumulation —
and is the checker of the CUDA kernel (csrc/arm_factor.cu). There is no
reference output to pin it against: it is checked for self-consistency —
FK orthonormality / reach / base-rotation equivariance and the
degenerate-covariance point cost (tests/test_arm.py), the Stein identity of the
moment-form gradients and the factorised-vs-joint ("Eq. 20") gradients of a
3-knot chain (tests/test_arm_cpu.py, the reference's test_factors.py:72-82 and
:136-162 restated for the arm potential).
"""

from __future__ import annotations

import numpy as np

from gvp_oracle import interp


def dh_transform(theta, d, a, alpha):
    """Standard Denavit-Hartenberg link transform Rz(theta) Tz(d) Tx(a) Rx(alpha)."""
    ct, st, ca, sa = np.cos(theta), np.sin(theta), np.cos(alpha), np.sin(alpha)
    return np.array([[ct, -st * ca, st * sa, a * ct],
                     [st, ct * ca, -ct * sa, a * st],
                     [0.0, sa, ca, d],
                     [0.0, 0.0, 0.0, 1.0]])


def link_frames(dh, base, q):
    """Frames 0..7 (4x4) of the arm at joint angles q. dh: (7, 4) rows
    (a, d, alpha, theta_offset)."""
    T = np.eye(4)
    T[:3, 3] = base
    frames = [T.copy()]
    for j in range(7):
        a, d, alpha, off = dh[j]
        T = T @ dh_transform(q[j] + off, d, a, alpha)
        frames.append(T.copy())
    return frames


def sphere_centers(dh, base, sphere_link, sphere_geom, q):
    frames = link_frames(dh, base, q)
    out = np.empty((len(sphere_link), 3))
    for s, (lk, g) in enumerate(zip(sphere_link, sphere_geom)):
        F = frames[int(lk)]
        out[s] = F[:3, :3] @ g[:3] + F[:3, 3]
    return out


def arm_cost(dh, base, sphere_link, sphere_geom, grid, origin, cell, radius_eps, sigma_obs, q):
    """psi(q) and the number of out-of-bounds sphere centres."""
    c = sphere_centers(dh, base, sphere_link, sphere_geom, q)
    d, oob = interp(grid, origin, cell, c)
    gap = sphere_geom[:, 3] + radius_eps - d
    return float(sigma_obs * np.sum(np.where(gap > 0.0, gap * gap, 0.0))), oob


def arm_factor_expectations(means, chols, points, weights, grid, origin, cell, dh, base, sphere_link,
                            sphere_geom, radius_eps, sigma_obs):
    """e0 = sum_l w_l psi(x_l), e1 = sum_l w_l psi dx_l, e2 = sum_l w_l psi dx_l dx_l^T with
    x_l = mu + L xi_l (the reference's moment contract, _kernels.pyx:93-129), psi reading
    q = x[:7]. Returns (e0 (F,), e1 (F, n), e2 (F, n, n), oob)."""
    means = np.asarray(means, float)
    chols = np.asarray(chols, float)
    F, n = means.shape
    e0 = np.zeros(F)
    e1 = np.zeros((F, n))
    e2 = np.zeros((F, n, n))
    oob = 0
    for f in range(F):
        dx = points @ chols[f].T
        for l in range(len(weights)):
            psi, o = arm_cost(dh, base, sphere_link, sphere_geom, grid, origin, cell, radius_eps, sigma_obs,
                              means[f, :7] + dx[l, :7])
            oob += o
            if psi == 0.0:
                continue
            w = weights[l] * psi
            e0[f] += w
            e1[f] += w * dx[l]
            e2[f] += w * np.outer(dx[l], dx[l])
    return e0, e1, e2, oob


def arm_evaluate_factors(mean, covs, points, weights, grid, origin, cell, dh, base, sphere_link, sphere_geom,
                         radius_eps, sigma_obs):
    """The factor stage (factors.py:167-225) with the arm potential: interior
    knots 1..K-2, gaussian_sqrt roots, moments, _moment_gradients; returns
    (e_psi (F,), g_mu (F, n), g_sigma (F, n, n), oob)."""
    from gvp_oracle import gaussian_sqrt, moment_gradients

    mean = np.asarray(mean, float)
    covs = np.asarray(covs, float)
    K, n = mean.shape
    F = max(K - 2, 0)
    chols = np.stack([gaussian_sqrt(covs[i]) for i in range(1, K - 1)]) if F else np.zeros((0, n, n))
    e0, e1, e2, oob = arm_factor_expectations(mean[1:K - 1], chols, points, weights, grid, origin, cell, dh, base,
                                              sphere_link, sphere_geom, radius_eps, sigma_obs)
    g_mu, g_s = np.zeros((F, n)), np.zeros((F, n, n))
    for f in range(F):
        g_mu[f], g_s[f] = moment_gradients(e0[f], e1[f], e2[f], covs[f + 1])
    return np.maximum(e0, 0.0), g_mu, g_s, oob
