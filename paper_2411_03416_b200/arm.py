"""7-DOF sphere-arm collision factor (configuration C3).

The reference's factor expectation (`_kernels.pyx:93-129`) for a manipulator
whose body is covered by spheres on its links: psi(q) = sigma * sum_s
max(r_s + eps - d(FK_s(q)), 0)^2 with q the 7 joint angles (state (q, q_dot),
n = 14) and d the reference's trilinear SDF. The reference has no such model;
the CPU oracle `oracle/arm_oracle.py` restates this definition and the CUDA
kernel `csrc/arm_factor.cu` is checked against it (parity unpinned by a
reference, see the oracle's header).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .quadrature import QuadratureRule
from .sdf import CollisionModel, SignedDistanceField

NQ = 7


@dataclass(frozen=True)
class SphereArm:
    """Standard-DH 7-joint arm: dh rows (a, d, alpha, theta_offset) per joint;
    sphere s sits at `sphere_local[s]` in the frame after joint `sphere_link[s]`
    (0 = base frame) with radius `sphere_radius[s]`."""

    dh: np.ndarray
    base: np.ndarray
    sphere_link: np.ndarray
    sphere_local: np.ndarray
    sphere_radius: np.ndarray

    def __post_init__(self):
        dh = np.asarray(self.dh, dtype=np.float64).reshape(NQ, 4)
        link = np.asarray(self.sphere_link, dtype=np.int32).reshape(-1)
        loc = np.asarray(self.sphere_local, dtype=np.float64).reshape(-1, 3)
        rad = np.asarray(self.sphere_radius, dtype=np.float64).reshape(-1)
        if not (len(link) == len(loc) == len(rad)):
            raise ValueError("sphere tables must align")
        if np.any(link < 0) or np.any(link > NQ):
            raise ValueError("sphere_link must be in 0..7")
        object.__setattr__(self, "dh", dh)
        object.__setattr__(self, "base", np.asarray(self.base, dtype=np.float64).reshape(3))
        object.__setattr__(self, "sphere_link", link)
        object.__setattr__(self, "sphere_local", loc)
        object.__setattr__(self, "sphere_radius", rad)

    @property
    def geom(self) -> np.ndarray:
        return np.concatenate([self.sphere_local, self.sphere_radius[:, None]], axis=1)


def panda_like(base=(0.0, 0.0, 0.0)) -> SphereArm:
    """A Franka-Panda-sized arm in standard DH with two spheres per moving link."""
    dh = np.array([[0.0, 0.333, -np.pi / 2, 0.0],
                   [0.0, 0.0, np.pi / 2, 0.0],
                   [0.0825, 0.316, np.pi / 2, 0.0],
                   [-0.0825, 0.0, -np.pi / 2, 0.0],
                   [0.0, 0.384, np.pi / 2, 0.0],
                   [0.088, 0.0, np.pi / 2, 0.0],
                   [0.0, 0.107, 0.0, 0.0]])
    link, loc, rad = [], [], []
    for j in range(1, NQ + 1):
        for z in (-0.06, 0.0):
            link.append(j)
            loc.append((0.0, 0.0, z))
            rad.append(0.08 if j < 6 else 0.06)
    return SphereArm(dh=dh, base=np.asarray(base, float), sphere_link=np.array(link), sphere_local=np.array(loc),
                     sphere_radius=np.array(rad))


@dataclass
class ArmProjection:
    """Distinct joint-space projections xi[:7] of a rule and their weight
    moments [m0 | m1 (n) | m2 (n(n+1)/2, packed lower)]."""

    proj: np.ndarray
    mom: np.ndarray
    cnt: np.ndarray


def arm_projection_tables(rule: QuadratureRule) -> ArmProjection:
    pts, w = np.asarray(rule.points, float), np.asarray(rule.weights, float)
    n = pts.shape[1]
    if n != 2 * NQ:
        raise ValueError(f"the arm state is (q, q_dot): n = {2 * NQ}, rule has {n}")
    keys, inv = np.unique(pts[:, :NQ], axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    r, c = np.tril_indices(n)
    mom = np.zeros((len(keys), 1 + n + len(r)))
    cnt = np.zeros(len(keys), dtype=np.int32)
    for l in range(len(w)):
        j = inv[l]
        mom[j, 0] += w[l]
        mom[j, 1:1 + n] += w[l] * pts[l]
        mom[j, 1 + n:] += w[l] * (pts[l][:, None] * pts[l][None, :])[r, c]
        cnt[j] += 1
    return ArmProjection(proj=np.ascontiguousarray(keys), mom=mom, cnt=cnt)


def arm_factor_expectations(means, chols, rule: QuadratureRule, sdf: SignedDistanceField, arm: SphereArm,
                            model: CollisionModel, tables: ArmProjection | None = None):
    """(e0 (F,), e1 (F, 14), e2 (F, 14, 14), oob) for F factors on the GPU."""
    if sdf.values.ndim != 3:
        raise ValueError("the arm needs a 3D signed-distance field")
    tab = tables or arm_projection_tables(rule)
    means = N.f64(means)
    chols = N.f64(chols)
    F = means.shape[0]
    e0, e1, e2 = np.empty(F), np.empty((F, 2 * NQ)), np.empty((F, 2 * NQ, 2 * NQ))
    oob = np.zeros(1, dtype=np.int64)
    grid = N.f64(sdf.values)
    code = N.load().gvp_arm_factor_expectations(
        F, N.ptr(means), N.ptr(chols), len(tab.proj), N.ptr(N.f64(tab.proj)), N.ptr(N.f64(tab.mom)),
        N.ptr(np.ascontiguousarray(tab.cnt, dtype=np.int32)), N.ptr(grid),
        N.ptr(np.asarray(grid.shape, dtype=np.int64)), N.ptr(N.f64(sdf.origin)), float(sdf.cell_size),
        N.ptr(N.f64(arm.dh)), N.ptr(N.f64(arm.base)), len(arm.sphere_link),
        N.ptr(np.ascontiguousarray(arm.sphere_link, dtype=np.int32)), N.ptr(N.f64(arm.geom)),
        float(model.radius_eps), float(model.sigma_obs), N.ptr(e0), N.ptr(e1), N.ptr(e2), N.ptr(oob))
    N.check(code, "gvp_arm_factor_expectations")
    if code != N.GVP_OK:
        raise RuntimeError(f"gvp_arm_factor_expectations: {N.last_error()}")
    return e0, e1, e2, int(oob[0])


class ArmEnvironment:
    """Collision environment of the 7-DOF sphere arm for ``run_pgvimp`` (the
    reference's ``Environment(sdf, model)`` with the arm's forward kinematics):
    the 3D map, the arm and the rule's projection tables stay resident on the
    device (gvp_arm_create); every factor stage is one call
    (gvp_arm_factor_grads: gaussian_sqrt -> moments -> moment gradients)."""

    def __init__(self, sdf: SignedDistanceField, model: CollisionModel, arm: SphereArm):
        if sdf.values.ndim != 3:
            raise ValueError("the arm needs a 3D signed-distance field")
        self.sdf, self.model, self.arm = sdf, model, arm
        self._handle = None
        self._rule_id = None

    def _bind(self, rule: QuadratureRule):
        if self._handle is not None and self._rule_id == id(rule):
            return self._handle
        self.close()
        tab = arm_projection_tables(rule)
        grid = N.f64(self.sdf.values)
        h = N.C.c_void_p()
        lib = N.load()
        code = lib.gvp_arm_create(
            N.C.byref(h), N.ptr(grid), N.ptr(np.asarray(grid.shape, dtype=np.int64)), N.ptr(N.f64(self.sdf.origin)),
            float(self.sdf.cell_size), N.ptr(N.f64(self.arm.dh)), N.ptr(N.f64(self.arm.base)),
            len(self.arm.sphere_link), N.ptr(np.ascontiguousarray(self.arm.sphere_link, dtype=np.int32)),
            N.ptr(N.f64(self.arm.geom)), float(self.model.radius_eps), float(self.model.sigma_obs), len(tab.proj),
            N.ptr(N.f64(tab.proj)), N.ptr(N.f64(tab.mom)), N.ptr(np.ascontiguousarray(tab.cnt, dtype=np.int32)))
        N.check(code, "gvp_arm_create")
        if code != N.GVP_OK:
            raise RuntimeError(f"gvp_arm_create: {N.last_error()}")
        self._handle, self._rule_id, self._rule = h, id(rule), rule
        return h

    def factor_gradients(self, joint_mean, covs, rule: QuadratureRule):
        """(e_psi (F,), g_mu (F, 14), g_sigma (F, 14, 14)) of the interior
        knots 1..K-2 (factors.py:159-225 with the arm's potential)."""
        from .factors import FactorEvaluationError

        covs = np.asarray(covs, dtype=np.float64)
        K = covs.shape[0]
        mean = np.asarray(joint_mean, dtype=np.float64).reshape(K, 2 * NQ)
        F = max(K - 2, 0)
        e_psi, g_mu, g_s = np.zeros(F), np.zeros((F, 2 * NQ)), np.zeros((F, 2 * NQ, 2 * NQ))
        if F == 0:
            return e_psi, g_mu, g_s
        h = self._bind(rule)
        oob, where = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
        code = N.load().gvp_arm_factor_grads(h, F, N.ptr(N.f64(mean[1:K - 1])), N.ptr(N.f64(covs[1:K - 1])),
                                             N.ptr(e_psi), N.ptr(g_mu), N.ptr(g_s), N.ptr(oob), N.ptr(where))
        N.check(code, "gvp_arm_factor_grads")
        if code == N.GVP_ERR_NONFINITE:
            raise FactorEvaluationError(int(where[0]) + 1, "non-finite expectation")
        if code == N.GVP_ERR_SQRT:
            raise NotImplementedError(f"factor {int(where[0]) + 1}: covariance needs the eigh root of gaussian_sqrt")
        if code != N.GVP_OK:
            raise RuntimeError(f"gvp_arm_factor_grads: {N.last_error()}")
        self.sdf.note_oob(int(oob[0]))
        return e_psi, g_mu, g_s

    def close(self):
        if self._handle is not None:
            N.load().gvp_arm_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def joint_double_integrator(nsteps: int, dt: float):
    """Joint-space double integrator of the 7-DOF arm (the point_robot_lti
    construction of dynamics.py:66-87 at 7 joints): state (q, q_dot), n = 14,
    A = [[0, I], [0, 0]], a = 0, B = [0; I]."""
    from .dynamics import LTVStep, LTVSystem

    A = np.zeros((2 * NQ, 2 * NQ))
    A[:NQ, NQ:] = np.eye(NQ)
    B = np.zeros((2 * NQ, NQ))
    B[NQ:, :] = np.eye(NQ)
    step = LTVStep(A=A, a=np.zeros(2 * NQ), B=B)
    return LTVSystem(steps=tuple([step] * (nsteps + 1)), dt=dt, n=2 * NQ, m=NQ)
