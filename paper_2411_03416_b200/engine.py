"""Host handle of the batched device engine (csrc/engine.cu).

``PlanBatch`` owns one ``gvp_engine``: B independent P-GVIMP problems on one
GPU sharing an SDF and a quadrature rule, all state resident in HBM in the
plan-minor layout (include/gvp_b200.h). Arrays cross this API batch-major,
shape (B, K, ...); the transposition to plan-minor happens here.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .quadrature import QuadratureRule
from .sdf import CollisionModel, SignedDistanceField

RECORD_KEYS = ("beta", "temperature", "prior_cost", "collision_cost", "entropy_cost",
               "total_cost", "kl_step", "mean_shift")


def to_plan_minor(x: np.ndarray) -> np.ndarray:
    """(B, ...) -> (..., B) C-contiguous."""
    return np.ascontiguousarray(np.moveaxis(np.asarray(x, dtype=np.float64), 0, -1))


def from_plan_minor(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.moveaxis(x, -1, 0))


_FAR_FIELD = None


def far_field() -> SignedDistanceField:
    """Obstacle-free stand-in (env=None): every hinge is exactly zero."""
    global _FAR_FIELD
    if _FAR_FIELD is None:
        _FAR_FIELD = SignedDistanceField(origin=np.zeros(2), cell_size=1.0, values=np.full((2, 2), 1e6))
    return _FAR_FIELD


class PlanBatch:
    def __init__(self, nplans: int, nknots: int, n: int, sdf: SignedDistanceField,
                 model: CollisionModel, rule: QuadratureRule, cfg, shared_prior: bool = True,
                 spec_lanes: int = 0):
        self.lib = N.load()
        self.B, self.K, self.n = int(nplans), int(nknots), int(n)
        self.shared_prior = bool(shared_prior)
        self.max_iters = int(cfg.max_iters)
        c = N.PlanConfig(kl_bound=cfg.kl_bound, beta_min=cfg.beta_min, beta_max=cfg.beta_max,
                         temp_low=cfg.temp_low, temp_high=cfg.temp_high,
                         collision_tol=-1.0 if cfg.collision_tol is None else cfg.collision_tol,
                         tol_mean=cfg.tol_mean, tol_cost=cfg.tol_cost,
                         init_cov_scale=cfg.init_cov_scale, max_iters=cfg.max_iters,
                         spec_lanes=spec_lanes)
        self._cfg = c
        h = C.c_void_p()
        grid = N.f64(sdf.values)
        self._grid_dim = grid.ndim
        shape = np.asarray(grid.shape, dtype=np.int64)
        origin = N.f64(sdf.origin)
        code = self.lib.gvp_engine_create(C.byref(h), self.B, self.K, self.n, int(self.shared_prior),
                                          N.ptr(grid), grid.ndim, N.ptr(shape), N.ptr(origin),
                                          float(sdf.cell_size), float(model.radius_eps),
                                          float(model.sigma_obs), N.ptr(rule.points),
                                          N.ptr(rule.weights), rule.npoints, C.byref(c))
        N.check(code, "gvp_engine_create")
        if code != N.GVP_OK:
            raise RuntimeError(f"gvp_engine_create: {N.last_error()}")
        self.handle = h

    # ------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "handle", None):
            self.lib.gvp_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, code, what):
        N.check(code, what)
        if code != N.GVP_OK:
            raise RuntimeError(f"{what}: {N.last_error()}")

    # ------------------------------------------------------------ problem
    def load(self, kdiag, koff, info, prior_mean, init_mean):
        """kdiag (K,n,n)/koff (K-1,n,n) if shared_prior else (B,K,n,n)/(B,K-1,n,n);
        info, prior_mean, init_mean (B, K, n)."""
        if self.shared_prior:
            kd, ko = N.f64(kdiag), N.f64(koff)
        else:
            kd, ko = to_plan_minor(kdiag), to_plan_minor(koff)
        inf, pm, m0 = to_plan_minor(info), to_plan_minor(prior_mean), to_plan_minor(init_mean)
        self._ok(self.lib.gvp_engine_load(self.handle, N.ptr(kd), N.ptr(ko), N.ptr(inf), N.ptr(pm),
                                          N.ptr(m0)), "gvp_engine_load")

    def load_boundary(self, kdiag, koff, base_info, base_mean, resp0, respg, anchor, x0s, goals):
        """A shared-prior batch by its boundary states (optimizer.batch_parts):
        plan 0's prior blocks / info / mean, the responses (n, K, n) and anchor
        (n, n), every plan's start and goal (B, n); the per-plan information,
        prior mean and straight-line initial mean are formed on the device."""
        a = [N.f64(x) for x in (kdiag, koff, base_info, base_mean, resp0, respg, anchor, x0s, goals)]
        self._ok(self.lib.gvp_engine_load_boundary(self.handle, *[N.ptr(x) for x in a]),
                 "gvp_engine_load_boundary")

    def load_device(self, kdiag_ptr, koff_ptr, info_ptr, pmean_ptr, mean_ptr):
        """Device pointers already in the plan-minor layout (no host traffic)."""
        self._ok(self.lib.gvp_engine_load_dev(self.handle, kdiag_ptr, koff_ptr, info_ptr,
                                              pmean_ptr, mean_ptr), "gvp_engine_load_dev")

    # ------------------------------------------------------------ execution
    def step(self, iters: int = 1, sync: bool = False):
        self._ok(self.lib.gvp_engine_step(self.handle, int(iters), int(sync)), "gvp_engine_step")

    def step_beta(self, beta):
        """One iteration (synchronous) in which plan b takes step size beta[b]
        where it is finite (NaN: the searched one). The search still runs and
        is traced (`probes`), so a known step sequence can be replayed while
        every search is compared against it."""
        b = np.ascontiguousarray(np.asarray(beta, dtype=np.float64).reshape(-1))
        if b.shape != (self.B,):
            raise ValueError(f"beta needs {self.B} entries")
        self._ok(self.lib.gvp_engine_step_beta(self.handle, N.ptr(b)), "gvp_engine_step_beta")

    def set_state(self, plans, mean, diag, off):
        """Replace the iterate of the given plans (batch-major over `plans`:
        mean (s, K, n), diag (s, K, n, n), off (s, K-1, n, n)) and recompute
        the marginals, log det and factor stage at it."""
        pl = np.ascontiguousarray(np.asarray(plans, dtype=np.int32).reshape(-1))
        s, K, n = len(pl), self.K, self.n
        m, d, o = N.f64(np.reshape(mean, (s, K, n))), N.f64(np.reshape(diag, (s, K, n, n))), \
            N.f64(np.reshape(off, (s, K - 1, n, n)))
        self._ok(self.lib.gvp_engine_set_state(self.handle, s, N.ptr(pl), N.ptr(m), N.ptr(d), N.ptr(o)),
                 "gvp_engine_set_state")

    def oob(self) -> np.ndarray:
        """Per-plan count of sigma points clamped at the SDF border so far."""
        out = np.zeros(self.B, dtype=np.int64)
        self._ok(self.lib.gvp_engine_get_oob(self.handle, N.ptr(out)), "gvp_engine_get_oob")
        return out

    def step_profiled(self, iters: int = 1) -> np.ndarray:
        """Kernel-by-kernel iterations with CUDA events; returns summed device
        ms of (bisection incl. the residual kernel, commit, factor kernel,
        eigh fix-up + control)."""
        ms = np.zeros(4)
        self._ok(self.lib.gvp_engine_step_profiled(self.handle, int(iters), N.ptr(ms)),
                 "gvp_engine_step_profiled")
        return ms

    PROFILE_BUCKETS = ("residual", "probes", "commit", "factor_grads", "eigh_fixup", "control")

    def step_profiled_ex(self, iters: int = 1) -> np.ndarray:
        """Same, one bucket per kernel (PROFILE_BUCKETS)."""
        ms = np.zeros(len(self.PROFILE_BUCKETS))
        self._ok(self.lib.gvp_engine_step_profiled_ex(self.handle, int(iters), N.ptr(ms), len(ms)),
                 "gvp_engine_step_profiled_ex")
        return ms

    def stream_ptr(self) -> int:
        return int(self.lib.gvp_engine_stream(self.handle) or 0)

    def sync(self):
        self._ok(self.lib.gvp_engine_sync(self.handle), "gvp_engine_sync")

    def active(self) -> int:
        out = np.zeros(1, dtype=np.int32)
        self._ok(self.lib.gvp_engine_active(self.handle, N.ptr(out)), "gvp_engine_active")
        return int(out[0])

    def run(self, check_every: int = 8) -> int:
        """Iterate until every plan stopped (converged, failed or max_iters)."""
        done = 0
        while done < self.max_iters:
            k = min(check_every, self.max_iters - done)
            self.step(k)
            done += k
            if self.active() == 0:
                break
        self.sync()
        return done

    def lanes(self) -> int:
        return int(self.lib.gvp_engine_lanes(self.handle))

    def launches(self) -> int:
        return int(self.lib.gvp_engine_launches(self.handle))

    def set_map_bank(self, maps, plan_map):
        """Per-plan signed-distance maps: `maps` is a sequence of
        SignedDistanceField (or raw value arrays) with the engine's grid
        geometry; plan b reads maps[plan_map[b]]. Call before stepping."""
        vals = [np.asarray(getattr(m, "values", m), dtype=np.float64) for m in maps]
        grids = N.f64(np.stack(vals))
        pm = np.ascontiguousarray(np.asarray(plan_map, dtype=np.int32))
        if pm.shape != (self.B,):
            raise ValueError(f"plan_map needs {self.B} entries")
        self._ok(self.lib.gvp_engine_set_map_bank(self.handle, len(vals), N.ptr(grids), N.ptr(pm)),
                 "gvp_engine_set_map_bank")

    def raster_map_bank(self, primitive_lists, plan_map):
        """Map bank rasterised on the device from primitive lists (one list of
        Disc/Box per map, rasterize semantics on the engine's grid)."""
        from .sdf import primitive_table

        dim = self._grid_dim
        off = np.zeros(len(primitive_lists) + 1, dtype=np.int32)
        kinds, params = [], []
        for m, prims in enumerate(primitive_lists):
            k, p = primitive_table(list(prims), dim)
            kinds.append(k)
            params.append(p)
            off[m + 1] = off[m] + len(prims)
        kinds = np.ascontiguousarray(np.concatenate(kinds) if kinds else np.zeros(0, np.int32), dtype=np.int32)
        params = N.f64(np.concatenate(params) if params else np.zeros((0, 2 * dim)))
        pm = np.ascontiguousarray(np.asarray(plan_map, dtype=np.int32))
        if pm.shape != (self.B,):
            raise ValueError(f"plan_map needs {self.B} entries")
        self._ok(self.lib.gvp_engine_raster_map_bank(self.handle, len(primitive_lists), N.ptr(off), N.ptr(kinds),
                                                     N.ptr(params), N.ptr(pm)), "gvp_engine_raster_map_bank")

    def trace_probes(self, max_probes: int = 64):
        """Record each plan's step-size probes (optimizer.py:188-231 `trace`);
        call before the first step."""
        self._ok(self.lib.gvp_engine_trace_probes(self.handle, int(max_probes)), "gvp_engine_trace_probes")
        self._max_probes = int(max_probes)

    def probes(self):
        """Last iteration's probes per plan: list of (n_i, 3) arrays of
        (beta, spd, kl) in the reference's probe order."""
        log = np.empty((self.B, self._max_probes, 3))
        cnt = np.zeros(self.B, dtype=np.int32)
        self._ok(self.lib.gvp_engine_get_probes(self.handle, N.ptr(log), N.ptr(cnt)), "gvp_engine_get_probes")
        return [log[b, :min(int(cnt[b]), self._max_probes)] for b in range(self.B)]

    # ------------------------------------------------------------ results
    def state(self):
        B, K, n = self.B, self.K, self.n
        mean = np.empty((K, n, B))
        diag = np.empty((K, n, n, B))
        off = np.empty((K - 1, n, n, B))
        covs = np.empty((K, n, n, B))
        crosses = np.empty((K - 1, n, n, B))
        self._ok(self.lib.gvp_engine_get_state(self.handle, N.ptr(mean), N.ptr(diag), N.ptr(off),
                                               N.ptr(covs), N.ptr(crosses)), "gvp_engine_get_state")
        return {"mean": from_plan_minor(mean), "diag": from_plan_minor(diag),
                "off": from_plan_minor(off), "covs": from_plan_minor(covs),
                "crosses": from_plan_minor(crosses)}

    def packed_into(self, mean=None, covs=None):
        """Fetch into caller buffers without host unpacking (pinned buffers
        make this a straight DMA): mean (K, n, B) plan-minor, covs packed
        lower-symmetric (K, n(n+1)/2, B)."""
        for a, shape in ((mean, (self.K, self.n, self.B)), (covs, (self.K, self.n * (self.n + 1) // 2, self.B))):
            if a is not None and (a.shape != shape or a.dtype != np.float64 or not a.flags.c_contiguous):
                raise ValueError(f"buffer must be C-contiguous float64 {shape}")
        self._ok(self.lib.gvp_engine_get_packed(self.handle, N.ptr(mean), N.ptr(covs)), "gvp_engine_get_packed")

    def mean(self) -> np.ndarray:
        """Joint means only, (B, K, n)."""
        m = np.empty((self.K, self.n, self.B))
        self._ok(self.lib.gvp_engine_get_state(self.handle, N.ptr(m), None, None, None, None),
                 "gvp_engine_get_state")
        return from_plan_minor(m)

    def summary(self):
        B = self.B
        arrs = [np.zeros(B, dtype=np.int32) for _ in range(5)]
        self._ok(self.lib.gvp_engine_get_summary(self.handle, *[N.ptr(a) for a in arrs]),
                 "gvp_engine_get_summary")
        return dict(zip(("converged", "iterations", "switch_iteration", "status", "where"), arrs))

    def records(self) -> np.ndarray:
        """(B, max_iters, 8) in RECORD_KEYS order; NaN past each plan's end."""
        rec = np.empty((self.max_iters, self.B, N.GVP_NREC))
        self._ok(self.lib.gvp_engine_get_records(self.handle, N.ptr(rec)), "gvp_engine_get_records")
        return np.ascontiguousarray(np.moveaxis(rec, 1, 0))

    def device_state(self):
        ptrs = [C.c_void_p() for _ in range(5)]
        self._ok(self.lib.gvp_engine_device_state(self.handle, *[C.byref(p) for p in ptrs]),
                 "gvp_engine_device_state")
        return dict(zip(("mean", "diag", "off", "covs", "crosses"), [p.value for p in ptrs]))
