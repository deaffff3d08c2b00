"""Result / cost-log / bench-CSV formats (runio.py) against
the reference's own writers and readers (oracle/_ref)."""

import json
import os
import sys
import types

import numpy as np
import pytest

from conftest import golden, rel_err

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _ref_runio():
    if not os.path.isdir(os.path.join(REF, "gvplan")):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, REF)
    try:
        from gvplan import runio as R
        from gvplan import bench as RB
    finally:
        sys.path.remove(REF)
    return R, RB


def _fake_result(rng, K=6, n=4, iters=3):
    covs = []
    for _ in range(K):
        a = rng.normal(size=(n, n))
        covs.append(a @ a.T + n * np.eye(n))
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    recs = [dict({"type": "iter", "iter": i + 1}, **{k: float(rng.normal()) for k in keys}) for i in range(iters)]
    final = types.SimpleNamespace(block_size=n, mean=rng.normal(size=K * n))
    return types.SimpleNamespace(final=final, marginals=types.SimpleNamespace(covs=covs), records=recs,
                                 converged=True, iterations=iters, switch_iteration=2)


def test_result_json_byte_identical_to_reference(tmp_path):
    from paper_2411_03416_b200 import runio

    R, _ = _ref_runio()
    res = _fake_result(np.random.default_rng(5))
    ours = runio.result_payload(res, "point2d", 2, 7, min_clear=0.25, mode="batch")
    ref = R.result_payload(res, "point2d", 2, 7, min_clear=0.25, mode="batch")
    assert json.dumps(ours, sort_keys=True) == json.dumps(ref, sort_keys=True)
    runio.write_result(str(tmp_path / "a.json"), ours)
    R.write_result(str(tmp_path / "b.json"), ref)
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    back = R.load_result(str(tmp_path / "a.json"))  # the reference reads our file
    assert all(np.allclose(a, b) for a, b in zip(R.result_marginals(back), res.marginals.covs))


def test_costs_jsonl_and_bench_csv_match_reference(tmp_path):
    from paper_2411_03416_b200 import runio

    R, RB = _ref_runio()
    res = _fake_result(np.random.default_rng(6))
    runio.write_costs_jsonl(str(tmp_path / "a.jsonl"), res.records, {"seed": 3})
    R.write_costs_jsonl(str(tmp_path / "b.jsonl"), res.records, {"seed": 3})
    assert (tmp_path / "a.jsonl").read_bytes() == (tmp_path / "b.jsonl").read_bytes()
    assert R.read_costs_jsonl(str(tmp_path / "a.jsonl")) == runio.read_costs_jsonl(str(tmp_path / "b.jsonl"))
    rows = [runio.bench_row("gpu", 1000, 4, 3, 4100.0, 14.9)]
    ref_rows = [RB._row("gpu", 1000, 4, 3, 4100.0, 14.9)]
    assert runio.rows_to_csv(rows) == RB.rows_to_csv(ref_rows)


def test_pack_roundtrip_and_schema_errors(tmp_path):
    from paper_2411_03416_b200 import runio

    a = np.random.default_rng(1).normal(size=(5, 5))
    s = a + a.T
    assert np.array_equal(runio.unpack_lower(runio.pack_lower(s), 5), s)
    with pytest.raises(ValueError):
        runio.unpack_lower([1.0, 2.0], 3)
    (tmp_path / "x.json").write_text(json.dumps({"schema": "other"}))
    with pytest.raises(ValueError):
        runio.load_result(str(tmp_path / "x.json"))


@pytest.mark.gpu
def test_gpu_run_writes_reference_readable_files(gpu, tmp_path):
    import paper_2411_03416_b200 as P

    R, _ = _ref_runio()
    g = golden("runs")
    sdf = P.rasterize([P.sdf.Disc(center=np.array([1.0, 0.75]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                      cell_size=0.05)
    env = P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=0.2, sigma_obs=8.0))
    res = P.run_pgvimp(P.point_robot_lti(2)(15, 0.2), env, P.OptimizerConfig(max_iters=25), np.zeros(4),
                       np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    clear = P.min_clearance(res.final.mean.reshape(16, 4), sdf, env.model)
    P.write_result(str(tmp_path / "result.json"), P.result_payload(res, "point2d", 2, 0, min_clear=clear))
    P.write_costs_jsonl(str(tmp_path / "costs.jsonl"), res.records)
    back = R.load_result(str(tmp_path / "result.json"))
    assert rel_err(np.array(back["states"]), g["t15_final_mean"]) <= 1e-9
    assert rel_err(np.stack(R.result_marginals(back)), g["t15_final_covs"]) <= 1e-9
    recs = [r for r in R.read_costs_jsonl(str(tmp_path / "costs.jsonl")) if r.get("type") == "iter"]
    assert [r["beta"] for r in recs] == list(g["t15_records"][:, 0])


@pytest.mark.gpu
def test_batch_writer_one_payload_per_plan(gpu, tmp_path):
    import paper_2411_03416_b200 as P

    R, _ = _ref_runio()
    sdf = P.rasterize([P.sdf.Disc(center=np.array([1.0, 0.75]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                      cell_size=0.05)
    env = P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=0.2, sigma_obs=8.0))
    goals = np.array([[2.0, 1.5, 0, 0], [1.8, 1.6, 0, 0], [2.1, 1.2, 0, 0]])
    br = P.run_pgvimp_batch(P.point_robot_lti(2)(15, 0.2), env, P.OptimizerConfig(max_iters=10), np.zeros(4),
                            goals, 1.0, 1e-3)
    dirs = P.runio.write_batch(str(tmp_path), br, "point2d", 2, seeds=[0, 1, 2], meta={"batch": 3})
    assert len(dirs) == 3
    for b, d in enumerate(dirs):
        back = R.load_result(os.path.join(d, "result.json"))
        assert np.array_equal(np.array(back["states"]), br.mean[b])
        assert back["iterations"] == int(br.iterations[b]) and back["seed"] == b
        recs = R.read_costs_jsonl(os.path.join(d, "costs.jsonl"))
        assert recs[0]["type"] == "meta" and recs[0]["schema"] == "gvplan-costs-v1"
        assert len(recs) == 1 + int(br.iterations[b])
