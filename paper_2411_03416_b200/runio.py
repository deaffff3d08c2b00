"""Result and cost-log formats of the reference (`runio.py`, schemas
`gvplan-result-v1` / `gvplan-costs-v1`) for the GPU driver's results
(SURVEY.md §8-f2), plus the reference's bench CSV rows (`bench.py:26,130-139`).

The payloads carry the same keys, packing and key order as the reference's, so
`result.json` / `costs.jsonl` written here load with the reference's readers
and compare value by value with the oracle CLI's files. Batched runs
(`run_pgvimp_batch`, `PlanBatch`) get one payload per plan.
"""

from __future__ import annotations

import json
import os

import numpy as np

RESULT_SCHEMA = "gvplan-result-v1"
COSTS_SCHEMA = "gvplan-costs-v1"
BENCH_HEADER = "mode,N,n,k_q,serial_ms,parallel_ms,improvement_pct"
_FINAL_KEYS = ("prior_cost", "collision_cost", "entropy_cost", "total_cost")


def pack_lower(mat) -> list:
    """Lower triangle, row-major (runio.py:23-25)."""
    mat = np.asarray(mat, dtype=np.float64)
    r, c = np.tril_indices(mat.shape[0])
    return [float(x) for x in mat[r, c]]


def unpack_lower(packed, n: int) -> np.ndarray:
    """Inverse of pack_lower, symmetric (runio.py:28-37)."""
    out = np.zeros((n, n))
    r, c = np.tril_indices(n)
    vals = np.asarray(packed, dtype=np.float64)
    if vals.size != r.size:
        raise ValueError(f"packed block has {vals.size} entries, expected {r.size} for n={n}")
    out[r, c] = vals
    out[c, r] = vals
    return out


def _payload(states, covs, converged, iterations, switch_iteration, last_record, system, position_dim,
             seed, min_clear, mode):
    states = np.asarray(states, dtype=np.float64)
    n = states.shape[1]
    last = last_record or {}
    payload = {
        "schema": RESULT_SCHEMA,
        "system": system,
        "n": int(n),
        "num_knots": int(len(states)),
        "position_dim": int(position_dim),
        "seed": seed,
        "states": [[float(v) for v in row] for row in states],
        "cov_packing": "lower-row-major",
        "marginal_covs_packed": [pack_lower(c) for c in covs],
        "converged": bool(converged),
        "iterations": int(iterations),
        "switch_iteration": None if switch_iteration is None else int(switch_iteration),
        "final_costs": {k: last.get(k) for k in _FINAL_KEYS},
        "min_clearance": min_clear,
    }
    if mode is not None:
        payload["mode"] = mode
    return payload


def result_payload(result, system: str, position_dim: int, seed: int, min_clear: float | None = None,
                   mode: str | None = None) -> dict:
    """runio.py:40-73 for a RunResult of run_pgvimp / run_ipgvimp."""
    n = result.final.block_size
    return _payload(result.final.mean.reshape(-1, n), result.marginals.covs, result.converged,
                    result.iterations, result.switch_iteration,
                    result.records[-1] if result.records else None, system, position_dim, seed, min_clear,
                    mode)


def batch_payloads(batch, system: str, position_dim: int, seeds, min_clear=None, mode: str | None = None):
    """One result payload per plan of a BatchResult (run_pgvimp_batch)."""
    from .optimizer import RECORD_KEYS

    B = len(batch.iterations)
    seeds = np.broadcast_to(np.asarray(seeds), (B,))
    clear = np.broadcast_to(np.asarray(min_clear, dtype=object), (B,))
    out = []
    for b in range(B):
        it = int(batch.iterations[b])
        last = dict(zip(RECORD_KEYS, (float(v) for v in batch.records[b, it - 1]))) if it > 0 else None
        sw = int(batch.switch_iteration[b])
        out.append(_payload(batch.mean[b], batch.covs[b], batch.converged[b], it, None if sw < 0 else sw,
                            last, system, position_dim, int(seeds[b]), clear[b], mode))
    return out


def batch_records(batch, b: int) -> list:
    """The iteration records of plan b as the reference's record dicts."""
    from .optimizer import RECORD_KEYS

    recs = []
    for it in range(int(batch.iterations[b])):
        d = {"type": "iter", "iter": it + 1}
        d.update({k: float(v) for k, v in zip(RECORD_KEYS, batch.records[b, it])})
        recs.append(d)
    return recs


def write_result(path: str, payload: dict) -> None:
    """runio.py:76-79: indent 1, sorted keys, trailing newline."""
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=1, sort_keys=True)
        fh.write("\n")


def load_result(path: str) -> dict:
    with open(path) as fh:
        payload = json.load(fh)
    if payload.get("schema") != RESULT_SCHEMA:
        raise ValueError(f"{path}: unexpected schema {payload.get('schema')!r}")
    return payload


def result_marginals(payload: dict) -> list:
    n = payload["n"]
    return [unpack_lower(p, n) for p in payload["marginal_covs_packed"]]


def write_costs_jsonl(path: str, records: list, meta: dict | None = None) -> None:
    """runio.py:93-99: a meta line with the schema, then one record per line."""
    with open(path, "w") as fh:
        head = {"type": "meta", "schema": COSTS_SCHEMA}
        head.update(meta or {})
        fh.write(json.dumps(head) + "\n")
        for rec in records:
            fh.write(json.dumps(rec) + "\n")


def read_costs_jsonl(path: str) -> list:
    recs = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                recs.append(json.loads(line))
            except json.JSONDecodeError as exc:
                raise ValueError(f"{path}:{lineno}: invalid JSON ({exc})")
    return recs


def write_batch(directory: str, batch, system: str, position_dim: int, seeds, meta: dict | None = None,
                min_clear=None) -> list:
    """plan_<b>/result.json + plan_<b>/costs.jsonl for every plan; returns the paths."""
    paths = []
    for b, payload in enumerate(batch_payloads(batch, system, position_dim, seeds, min_clear)):
        d = os.path.join(directory, f"plan_{b:05d}")
        os.makedirs(d, exist_ok=True)
        write_result(os.path.join(d, "result.json"), payload)
        write_costs_jsonl(os.path.join(d, "costs.jsonl"), batch_records(batch, b), meta)
        paths.append(d)
    return paths


def bench_row(mode: str, n_intervals: int, n: int, k_q: int, serial_ms: float, parallel_ms: float) -> dict:
    """bench.py:29-39 (serial = reference CPU, parallel = this engine for the GPU rows)."""
    impr = 100.0 * (serial_ms - parallel_ms) / serial_ms if serial_ms > 0 else 0.0
    return {"mode": mode, "N": n_intervals, "n": n, "k_q": k_q, "serial_ms": serial_ms,
            "parallel_ms": parallel_ms, "improvement_pct": impr}


def rows_to_csv(rows: list) -> str:
    """bench.py:130-139, same header and number formats."""
    lines = [BENCH_HEADER]
    for r in rows:
        lines.append(f"{r['mode']},{r['N']},{r['n']},{r['k_q']},{r['serial_ms']:.3f},{r['parallel_ms']:.3f},"
                     f"{r['improvement_pct']:.2f}")
    return "\n".join(lines) + "\n"
