"""KL-proximal update loop (API of gvplan/optimizer.py), on the GPU.

* ``proximal_update``  -> gvp_proximal_update   (prox_update_kernel)
* ``select_step_size`` -> gvp_select_step_size  (select_step_kernel: the whole
                          bisection, each probe two fused chain passes)
* ``run_pgvimp``       -> the batched engine with B = 1 (csrc/engine.cu):
                          every iteration is one CUDA-graph replay of
                          step-select, factor stage and cost/convergence
                          control; nothing returns to the host until the
                          run stops.
* ``run_pgvimp_batch`` -> the same engine for many independent plans.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace, field

import numpy as np

from . import _native as N
from .blocktri import BlockTridiagonalMatrix, NotPositiveDefiniteError, logdet_block_tridiag
from .dynamics import LTVSystem
from .engine import RECORD_KEYS, PlanBatch, far_field
from .factors import FactorGradient, evaluate_all_factors
from .gbp import ChainMarginals, gbp_marginals, trace_product
from .prior import DiscretePrior, assemble_prior
from .quadrature import QuadratureRule, smolyak_rule
from .sdf import CollisionModel, SignedDistanceField

_LOG_2PI = float(np.log(2.0 * np.pi))
_BISECTION_RTOL = 1e-3


@dataclass(frozen=True)
class JointGaussian:
    mean: np.ndarray
    prec: BlockTridiagonalMatrix

    def __post_init__(self):
        mean = np.asarray(self.mean, dtype=np.float64).reshape(-1)
        if mean.shape[0] != self.prec.dim:
            raise ValueError(f"mean dim {mean.shape[0]} != precision dim {self.prec.dim}")
        object.__setattr__(self, "mean", mean)

    @property
    def nblocks(self) -> int:
        return self.prec.nblocks

    @property
    def block_size(self) -> int:
        return self.prec.block_size


@dataclass
class Environment:
    sdf: SignedDistanceField
    model: CollisionModel


@dataclass
class OptimizerConfig:
    """Defaults of optimizer.py:72-99."""

    kl_bound: float = 0.1
    beta_min: float = 1e-4
    beta_max: float = 0.9
    temp_low: float = 1.0
    temp_high: float = 10.0
    collision_tol: float | None = None
    max_iters: int = 200
    tol_mean: float = 1e-5
    tol_cost: float = 1e-6
    k_q: int = 3
    init: str = "interp"
    init_cov_scale: float = 0.1
    init_mean: np.ndarray | None = None
    threads: int = 1

    def validate(self) -> None:
        if self.kl_bound <= 0:
            raise ValueError("kl_bound must be positive")
        if not 0 < self.beta_min < self.beta_max:
            raise ValueError("need 0 < beta_min < beta_max")
        if self.temp_low <= 0 or self.temp_high <= 0:
            raise ValueError("temperatures must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.init not in ("interp", "flow", "prior"):
            raise ValueError("init must be 'interp', 'flow', or 'prior'")


@dataclass(frozen=True)
class CostBreakdown:
    prior_cost: float
    collision_cost: float
    entropy_cost: float

    @property
    def mp_cost(self) -> float:
        return self.prior_cost + self.collision_cost

    @property
    def total(self) -> float:
        return self.prior_cost + self.collision_cost + self.entropy_cost


@dataclass
class RunResult:
    final: JointGaussian
    marginals: ChainMarginals
    records: list = field(default_factory=list)
    converged: bool = False
    iterations: int = 0
    switch_iteration: int | None = None
    wall_time_ms: float = 0.0


@dataclass
class StepSelection:
    beta: float
    next_state: JointGaussian
    kl: float
    marginals: ChainMarginals
    probes: np.ndarray | None = None  # (nprobes, 3): beta, spd_ok, kl
    logdet: float | None = None       # log det of next_state.prec (None: not produced)


def _step_arrays(cur, prior, g_mu, g_sigma):
    K, n = cur.nblocks, cur.block_size
    return (N.f64(cur.mean).reshape(K, n), N.f64(cur.prec.diag_stack), N.f64(cur.prec.off_stack),
            N.f64(prior.prec.diag_stack), N.f64(prior.prec.off_stack), N.f64(prior.info).reshape(K, n),
            N.f64(g_mu).reshape(K, n), N.f64(g_sigma.diag_stack), N.f64(g_sigma.off_stack))


def proximal_update(cur: JointGaussian, prior: DiscretePrior, g_mu: np.ndarray,
                    g_sigma: BlockTridiagonalMatrix, beta: float, temp: float) -> JointGaussian:
    """One Theorem-1 step at step size beta (optimizer.py:129-161)."""
    if beta <= 0:
        raise ValueError("beta must be positive")
    lib = N.load()
    K, n = cur.nblocks, cur.block_size
    arrs = _step_arrays(cur, prior, g_mu, g_sigma)
    om, od, oo = np.empty((K, n)), np.empty((K, n, n)), np.empty((max(K - 1, 0), n, n))
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_proximal_update(*[N.ptr(a) for a in arrs], K, n, float(beta), float(temp),
                                           N.ptr(om), N.ptr(od), N.ptr(oo), N.ptr(where)),
                   "proximal_update")
    if code == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(f"pivot block {int(where[0])} is not positive definite")
    return JointGaussian(mean=om.reshape(-1), prec=BlockTridiagonalMatrix(od, oo))


def kl_joint(nxt: JointGaussian, cur: JointGaussian, nxt_marginals: ChainMarginals | None = None) -> float:
    """KL(next || cur), clipped at 0 (optimizer.py:164-177); marginals and
    log-dets from the GPU."""
    if nxt_marginals is None:
        nxt_marginals = gbp_marginals(nxt.prec)
    delta = cur.mean - nxt.mean
    val = 0.5 * (trace_product(cur.prec, nxt_marginals) + cur.prec.quad_form(delta) - cur.prec.dim
                 + logdet_block_tridiag(nxt.prec) - logdet_block_tridiag(cur.prec))
    return max(val, 0.0)


def select_step_size(cur: JointGaussian, prior: DiscretePrior, g_mu: np.ndarray,
                     g_sigma: BlockTridiagonalMatrix, cfg: OptimizerConfig, temp: float,
                     max_probes: int = 64, logdet_cur: float | None = None) -> StepSelection:
    """Largest feasible beta in [beta_min, beta_max] by bisection to 1e-3
    relative width (optimizer.py:188-231); the whole search runs on device.
    logdet_cur (optional): log det of cur.prec when the caller already has it
    (the previous step's `logdet`), saving a sweep; the result carries the
    accepted state's log det where the device path produces it."""
    lib = N.load()
    K, n = cur.nblocks, cur.block_size
    arrs = _step_arrays(cur, prior, g_mu, g_sigma)
    beta, kl, ld_next = np.zeros(1), np.zeros(1), np.full(1, np.nan)
    om, od, oo = np.empty((K, n)), np.empty((K, n, n)), np.empty((max(K - 1, 0), n, n))
    cv, cr = np.empty((K, n, n)), np.empty((max(K - 1, 0), n, n))
    plog = np.zeros((max_probes, 3))
    nprobes = np.zeros(1, dtype=np.int32)
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_select_step_size_ld(
        *[N.ptr(a) for a in arrs], K, n, float(temp), float(cfg.kl_bound), float(cfg.beta_min),
        float(cfg.beta_max), N.ptr(beta), N.ptr(kl), N.ptr(om), N.ptr(od), N.ptr(oo), N.ptr(cv),
        N.ptr(cr), N.ptr(plog), max_probes, N.ptr(nprobes), N.ptr(where),
        float("nan") if logdet_cur is None else float(logdet_cur), N.ptr(ld_next)), "select_step_size")
    if code == N.GVP_ERR_NO_FEASIBLE_STEP:
        raise RuntimeError(f"no feasible step size at beta_min={cfg.beta_min} (KL bound {cfg.kl_bound})")
    if code == N.GVP_ERR_NOT_SPD:
        w = int(where[0]) & ~N.GVP_WHERE_MEAN_SOLVE_BIAS
        raise NotPositiveDefiniteError(f"pivot block {w} is not positive definite")
    return StepSelection(beta=float(beta[0]),
                         next_state=JointGaussian(mean=om.reshape(-1), prec=BlockTridiagonalMatrix(od, oo)),
                         kl=float(kl[0]), marginals=ChainMarginals.from_stacks(cv, cr),
                         probes=plog[:min(int(nprobes[0]), max_probes)].copy(),
                         logdet=float(ld_next[0]) if np.isfinite(ld_next[0]) else None)


def entropy_of(prec: BlockTridiagonalMatrix) -> float:
    return 0.5 * (prec.dim * (_LOG_2PI + 1.0) - logdet_block_tridiag(prec))


def cost_breakdown(cur: JointGaussian, prior: DiscretePrior, temp: float,
                   marginals: ChainMarginals | None = None,
                   factor_values: list | None = None, env: Environment | None = None,
                   rule: QuadratureRule | None = None, threads: int = 1,
                   logdet: float | None = None) -> CostBreakdown:
    """(prior, collision, -T H) costs of an iterate (optimizer.py:238-277);
    logdet (optional): log det of cur.prec if the caller has it."""
    if marginals is None:
        marginals = gbp_marginals(cur.prec)
    delta = cur.mean - prior.mean
    prior_cost = 0.5 * prior.prec.quad_form(delta) + 0.5 * trace_product(prior.prec, marginals)
    if factor_values is None:
        if env is None:
            factor_values = []
        else:
            if rule is None:
                raise ValueError("rule required to evaluate collision cost")
            factor_values = evaluate_all_factors(cur.mean, cur.prec, env.sdf, env.model, rule,
                                                 threads=threads, marginals=marginals)
    if isinstance(factor_values, _StageArrays):  # same left-to-right float sum, no per-factor objects
        collision = float(sum(factor_values.e_psi.tolist()))
    else:
        collision = float(sum(f.e_psi for f in factor_values))
    return CostBreakdown(prior_cost=prior_cost, collision_cost=collision,
                         entropy_cost=-temp * (entropy_of(cur.prec) if logdet is None else
                                               0.5 * (cur.prec.dim * (_LOG_2PI + 1.0) - logdet)))


def initial_mean(prior: DiscretePrior, cfg: OptimizerConfig) -> np.ndarray:
    K, n = prior.nsteps + 1, prior.n
    if cfg.init_mean is not None:
        mean = np.asarray(cfg.init_mean, dtype=np.float64).reshape(-1)
        if mean.shape[0] != K * n:
            raise ValueError("init_mean has wrong dimension")
        return mean.copy()
    if cfg.init == "flow":
        return prior.flow_mean.copy()
    if cfg.init == "prior":
        return prior.mean.copy()
    a = np.linspace(0.0, 1.0, K).reshape(-1, 1)
    return ((1.0 - a) * prior.x0 + a * prior.goal).reshape(-1)


def initial_state(prior: DiscretePrior, cfg: OptimizerConfig) -> JointGaussian:
    """Sigma_0 = init_cov_scale K  <=>  Lambda_0 = K^{-1} / init_cov_scale
    (optimizer.py:280-296)."""
    return JointGaussian(mean=initial_mean(prior, cfg), prec=prior.prec.scaled(1.0 / cfg.init_cov_scale))


def _records_to_dicts(rec: np.ndarray, iters: int, ms_per_iter: float) -> list:
    out = []
    for it in range(iters):
        d = {"type": "iter", "iter": it + 1}
        d.update({k: float(v) for k, v in zip(RECORD_KEYS, rec[it])})
        d["wall_time_ms"] = ms_per_iter
        out.append(d)
    return out


def _raise_plan_status(status: int, where: int, cfg: OptimizerConfig):
    if status == N.GVP_ERR_NO_FEASIBLE_STEP:
        raise RuntimeError(f"no feasible step size at beta_min={cfg.beta_min} (KL bound {cfg.kl_bound})")
    if status == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(
            f"pivot block {where & ~N.GVP_WHERE_MEAN_SOLVE_BIAS} is not positive definite")
    if status == N.GVP_ERR_NONFINITE:
        from .factors import FactorEvaluationError
        raise FactorEvaluationError(where, "non-finite expectation")
    if status == N.GVP_ERR_SQRT:  # singular eigh root: np.linalg.solve in _moment_gradients (factors.py:98)
        raise np.linalg.LinAlgError(f"Singular matrix (factor {where}: eigh root of gaussian_sqrt)")
    if status != 0:
        raise RuntimeError(f"plan failed with status {status}")


class _StageArrays:
    """A device factor stage as arrays (e_psi (F,), g_mu (F, n), g_sigma (F, n, n))
    for the interior unary collision factors (factors.py:159-164): the host loop
    scatters them with block writes and cost_breakdown sums e_psi in factor
    order, without one FactorGradient object per factor."""

    __slots__ = ("e_psi", "g_mu", "g_sigma")

    def __init__(self, e_psi, g_mu, g_sigma):
        self.e_psi, self.g_mu, self.g_sigma = e_psi, g_mu, g_sigma

    def __len__(self):
        return len(self.e_psi)

    def __iter__(self):
        return (FactorGradient(e_psi=float(e), g_mu=gm, g_sigma=gs)
                for e, gm, gs in zip(self.e_psi, self.g_mu, self.g_sigma))

    def joint(self, K: int, n: int):
        """assemble_joint_gradients (factors.py:228-255) for factors 1..K-2: each
        block receives exactly one addend, added to the zero block in one sweep."""
        g_mu = np.zeros((K, n))
        g_mu[1:K - 1] += self.g_mu
        g_s = BlockTridiagonalMatrix.zeros(K, n)
        g_s.diag_stack[1:K - 1] += self.g_sigma
        return g_mu.reshape(-1), g_s


def _run_pgvimp_host(prior: DiscretePrior, env, cfg: OptimizerConfig, t0: float) -> RunResult:
    """Algorithm 1 (optimizer.py:299-401) as the reference's host loop, every
    kernel on the GPU: for block sizes the fused engine does not cover (the
    7-DOF arm's n = 14 runs on the wide-block chain kernels) and for the arm
    environment. Per iteration: factor stage, device bisection
    (select_step_size), factor stage of the accepted state, costs."""
    from .arm import ArmEnvironment
    from .factors import assemble_joint_gradients, evaluate_all_factors, interior_collision_maps

    K, n = prior.nsteps + 1, prior.n
    collision_tol = cfg.collision_tol if cfg.collision_tol is not None else 1e-4 * prior.nsteps
    rule = smolyak_rule(cfg.k_q, n) if env is not None else None
    maps = interior_collision_maps(K)

    def factors(joint: JointGaussian, marg: ChainMarginals):
        if isinstance(env, ArmEnvironment):
            e_psi, g_mu, g_s = env.factor_gradients(joint.mean, marg.covs_stack, rule)
            return _StageArrays(e_psi, g_mu, g_s)
        return evaluate_all_factors(joint.mean, joint.prec, env.sdf, env.model, rule, threads=cfg.threads,
                                    marginals=marg)

    cur = initial_state(prior, cfg)
    temp = cfg.temp_low
    result = RunResult(final=cur, marginals=gbp_marginals(cur.prec))
    prev_total = prev_temp = None
    switched = False
    cached = None
    ld_cur = None
    for it in range(1, cfg.max_iters + 1):
        t_iter = time.perf_counter()
        if env is not None:
            fv = cached if cached is not None else factors(cur, result.marginals)
            if isinstance(fv, _StageArrays):
                g_mu, g_sigma = fv.joint(K, n)
            else:
                g_mu, g_sigma = assemble_joint_gradients(fv, maps, K, n)
        else:
            g_mu, g_sigma = np.zeros(K * n), BlockTridiagonalMatrix.zeros(K, n)
        step = select_step_size(cur, prior, g_mu, g_sigma, cfg, temp, logdet_cur=ld_cur)
        ld_cur = step.logdet  # the next search's logdet_cur and this record's entropy
        nxt = step.next_state
        nxt_f = factors(nxt, step.marginals) if env is not None else []
        cached = nxt_f if env is not None else None
        costs = cost_breakdown(nxt, prior, temp, marginals=step.marginals, factor_values=nxt_f, logdet=ld_cur)
        mean_shift = float(np.linalg.norm(nxt.mean - cur.mean))
        result.records.append({"type": "iter", "iter": it, "beta": step.beta, "temperature": temp,
                               "prior_cost": costs.prior_cost, "collision_cost": costs.collision_cost,
                               "entropy_cost": costs.entropy_cost, "total_cost": costs.total,
                               "kl_step": step.kl, "mean_shift": mean_shift,
                               "wall_time_ms": (time.perf_counter() - t_iter) * 1e3})
        cur = nxt
        result.final, result.marginals, result.iterations = cur, step.marginals, it
        same_temp = prev_temp is not None and prev_temp == temp
        total_change = abs(costs.total - prev_total) if prev_total is not None else np.inf
        if same_temp and mean_shift < cfg.tol_mean and total_change < cfg.tol_cost:
            result.converged = True
            break
        prev_total = costs.total if same_temp or prev_temp is None else None
        prev_temp = temp
        if not switched and costs.collision_cost < collision_tol and temp != cfg.temp_high:
            temp = cfg.temp_high
            switched = True
            result.switch_iteration = it
            prev_total = None
    result.wall_time_ms = (time.perf_counter() - t0) * 1e3
    return result


def run_pgvimp(sys_ltv: LTVSystem, env: Environment | None, cfg: OptimizerConfig, x0, goal,
               q_c: float, sigma_b: float, prior: DiscretePrior | None = None,
               spec_lanes: int = 0) -> RunResult:
    """Algorithm 1 (optimizer.py:299-401) on the GPU engine (n in {2, 4, 6}
    with a planar/volumetric SDF); other block sizes and the 7-DOF arm
    environment run the reference's host loop over the device kernels."""
    from .arm import ArmEnvironment

    cfg.validate()
    t0 = time.perf_counter()
    if prior is None:
        prior = assemble_prior(sys_ltv, x0, goal, q_c, sigma_b)
    K, n = prior.nsteps + 1, prior.n
    if n not in (2, 4, 6) or isinstance(env, ArmEnvironment):
        return _run_pgvimp_host(prior, env, cfg, t0)
    rule = smolyak_rule(cfg.k_q, n)
    sdf = env.sdf if env is not None else far_field()
    model = env.model if env is not None else CollisionModel(0.0, 1.0)
    eng = PlanBatch(1, K, n, sdf, model, rule, cfg, shared_prior=True, spec_lanes=spec_lanes)
    try:
        eng.load(prior.prec.diag_stack, prior.prec.off_stack, prior.info.reshape(1, K, n),
                 prior.mean.reshape(1, K, n), initial_mean(prior, cfg).reshape(1, K, n))
        eng.run()
        st = eng.state()
        sm = eng.summary()
        rec = eng.records()[0]
        oob = int(eng.oob()[0])
    finally:
        eng.close()
    if env is not None:
        env.sdf.note_oob(oob)  # every factor stage's clamped points (factors.py:206)
    status, where = int(sm["status"][0]), int(sm["where"][0])
    _raise_plan_status(status, where, cfg)
    iters = int(sm["iterations"][0])
    wall = (time.perf_counter() - t0) * 1e3
    final = JointGaussian(mean=st["mean"][0].reshape(-1),
                          prec=BlockTridiagonalMatrix(st["diag"][0], st["off"][0]))
    sw = int(sm["switch_iteration"][0])
    return RunResult(final=final, marginals=ChainMarginals.from_stacks(st["covs"][0], st["crosses"][0]),
                     records=_records_to_dicts(rec, iters, wall / max(iters, 1)),
                     converged=bool(sm["converged"][0]), iterations=iters,
                     switch_iteration=None if sw < 0 else sw, wall_time_ms=wall)


@dataclass
class BatchResult:
    """Batch-major results of ``run_pgvimp_batch``."""

    mean: np.ndarray        # (B, K, n)
    diag: np.ndarray        # (B, K, n, n)
    off: np.ndarray         # (B, K-1, n, n)
    covs: np.ndarray
    crosses: np.ndarray
    records: np.ndarray     # (B, max_iters, 8), RECORD_KEYS
    converged: np.ndarray
    iterations: np.ndarray
    switch_iteration: np.ndarray
    status: np.ndarray
    wall_time_ms: float


def batch_parts(sys_ltv: LTVSystem, x0s, goals, q_c: float, sigma_b: float):
    """The shared part of a batch's priors (see batch_problem): plan 0's prior,
    the anchored-mean responses to unit start / goal offsets resp0 / respg
    (n, K, n), the anchor block, and the (B, n) starts and goals."""
    x0s = np.atleast_2d(np.asarray(x0s, dtype=np.float64))
    goals = np.atleast_2d(np.asarray(goals, dtype=np.float64))
    B = max(len(x0s), len(goals))
    x0s = np.ascontiguousarray(np.broadcast_to(x0s, (B, x0s.shape[1])))
    goals = np.ascontiguousarray(np.broadcast_to(goals, (B, goals.shape[1])))
    base = assemble_prior(sys_ltv, x0s[0], goals[0], q_c, sigma_b)
    K, n = base.nsteps + 1, base.n
    anchor = np.eye(n) / sigma_b ** 2
    from .prior import anchored_mean

    resp0, respg = np.zeros((n, K, n)), np.zeros((n, K, n))
    for j in range(n):
        e = np.zeros((K, n))
        e[0] = anchor[:, j]
        resp0[j] = anchored_mean(base.prec, e.reshape(-1)).reshape(K, n)
        e[0], e[-1] = 0.0, anchor[:, j]
        respg[j] = anchored_mean(base.prec, e.reshape(-1)).reshape(K, n)
    return base, resp0, respg, anchor, x0s, goals


def batch_problem(sys_ltv: LTVSystem, x0s, goals, q_c: float, sigma_b: float, cfg: OptimizerConfig):
    """The priors of B plans that share the system, q_c and sigma_b (SURVEY §8e
    batch axis) without B prior assemblies: the anchored precision does not
    depend on the boundary states, the information vector only at the two
    anchor knots (prior.py:140-150), and the anchored mean / flow are affine in
    them — so one prior (plan 0's) plus 2n unit responses of the mean solve
    (on the device) give every plan's. Returns (prior of plan 0, info (B,K,n),
    prior mean (B,K,n), initial mean (B,K,n))."""
    base, resp0, respg, anchor, x0s, goals = batch_parts(sys_ltv, x0s, goals, q_c, sigma_b)
    B, K, n = len(x0s), base.nsteps + 1, base.n
    d0, dg = x0s - x0s[0], goals - goals[0]
    info = np.repeat(base.info.reshape(1, K, n), B, axis=0)
    info[:, 0, :] += d0 @ anchor.T
    info[:, -1, :] += dg @ anchor.T
    pmean = (base.mean.reshape(1, K, n) + np.einsum("bj,jkn->bkn", d0, resp0)
             + np.einsum("bj,jkn->bkn", dg, respg))
    if cfg.init_mean is not None:
        init = np.repeat(initial_mean(base, cfg).reshape(1, K, n), B, axis=0)
    elif cfg.init not in ("flow", "prior"):  # initial_mean's straight line, every plan at once
        a = np.linspace(0.0, 1.0, K).reshape(1, K, 1)
        init = (1.0 - a) * x0s[:, None, :] + a * goals[:, None, :]
    elif cfg.init == "prior":
        init = pmean.copy()
    else:  # the flow is affine in x0: propagate the start offsets through the transitions
        flow = np.repeat(base.flow_mean.reshape(1, K, n), B, axis=0)
        dflow = d0.copy()
        for i in range(K - 1):
            dflow = dflow @ np.asarray(base.phis[i]).T
            flow[:, i + 1] += dflow
        flow[:, 0] += d0
        init = flow
    return base, info, pmean, init


def run_pgvimp_batch(sys_ltv: LTVSystem, env: Environment | None, cfg: OptimizerConfig, x0s, goals,
                     q_c: float, sigma_b: float, spec_lanes: int = 0) -> BatchResult:
    """Many independent plans on one GPU: same system, map and settings, per
    plan start/goal (SURVEY.md §8-e batch axis). Plans that fail are masked
    out with their status; the batch never aborts."""
    cfg.validate()
    t0 = time.perf_counter()
    line_init = cfg.init_mean is None and cfg.init not in ("flow", "prior")
    if line_init:  # the per-plan arrays are expanded on the device from the boundary states
        base, resp0, respg, anchor, x0a, goala = batch_parts(sys_ltv, x0s, goals, q_c, sigma_b)
        B, K, n = len(x0a), base.nsteps + 1, base.n
    else:
        base, info, pmean, init = batch_problem(sys_ltv, x0s, goals, q_c, sigma_b, cfg)
        B, K, n = info.shape
    rule = smolyak_rule(cfg.k_q, n)
    sdf = env.sdf if env is not None else far_field()
    model = env.model if env is not None else CollisionModel(0.0, 1.0)
    eng = PlanBatch(B, K, n, sdf, model, rule, cfg, shared_prior=True, spec_lanes=spec_lanes)
    try:
        if line_init:
            eng.load_boundary(base.prec.diag_stack, base.prec.off_stack, base.info, base.mean, resp0, respg,
                              anchor, x0a, goala)
        else:
            eng.load(base.prec.diag_stack, base.prec.off_stack, info, pmean, init)
        eng.run()
        st = eng.state()
        sm = eng.summary()
        rec = eng.records()
        oob = eng.oob()
    finally:
        eng.close()
    if env is not None:
        env.sdf.note_oob(int(oob.sum()))
    return BatchResult(records=rec, converged=sm["converged"].astype(bool),
                       iterations=sm["iterations"], switch_iteration=sm["switch_iteration"],
                       status=sm["status"], wall_time_ms=(time.perf_counter() - t0) * 1e3, **st)
