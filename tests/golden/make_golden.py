"""Generate golden fixtures by running the REAL reference (``baksolve`` 0.1.0).

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz
    python tests/golden/make_golden.py --bakp-only   # only the bakp_*.npz fixtures
    python tests/golden/make_golden.py --select-only # only the select_*.npz fixtures
    python tests/golden/make_golden.py --matio-only  # only the matio_* files (reference save_matrix)
    python tests/golden/make_golden.py --harness-only  # only harness_records.json (reference run_case)

The reference is imported from ``/root/reference/pkg/src`` (pure Python on
numpy/OpenBLAS).  Nothing at test time reads ``/root/reference``: the
fixtures committed next to this script carry everything the tests need.

Each fixture stores the solve inputs either explicitly (small, or built with
``np.random.default_rng`` as the reference's own tests do) or as a
``generate_system`` spec plus a SHA-256 of the drawn bytes (so the oracle's
generator restatement is pinned too), together with the reference's outputs:
a_hat, residual, per-sweep history, sweeps_run, converged, drift_warning,
and the fp64-recomputed residual norm of bench.py:180-184.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    sys.path.insert(0, REF_SRC)
    import baksolve as bk
    from baksolve.bench import _predict_f64
    from threadpoolctl import threadpool_info

    np.dot(np.ones(2), np.ones(2))
    blas = [i for i in threadpool_info() if i.get("user_api") == "blas"]
    host = {"numpy": np.__version__,
            "blas": (blas[0].get("internal_api"), blas[0].get("version"),
                     blas[0].get("architecture")) if blas else None}

    if "--select-only" in sys.argv:  # regenerate only the column-scoring / selection fixtures
        with open(os.path.join(HERE, "MANIFEST.json")) as f:
            man = json.load(f)
        man["select_cases"] = make_select(bk, host)
        with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
            json.dump(man, f, indent=1)
        return
    if "--harness-only" in sys.argv:  # regenerate only the run_case records
        make_harness(bk)
        return
    if "--matio-only" in sys.argv:  # regenerate only the BAKM / CSV files
        make_matio(bk)
        return
    if "--bakp-only" in sys.argv:  # regenerate only the blocked-solver fixtures
        with open(os.path.join(HERE, "MANIFEST.json")) as f:
            man = json.load(f)
        man["bakp_cases"] = make_bakp(bk, host, _predict_f64)
        with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
            json.dump(man, f, indent=1)
        return

    cases = []

    def add(name, x, y, cfg, a0=None, spec=None, store_inputs=True):
        rep = bk.solve_bak(x, y, cfg, a0=a0)
        pred = _predict_f64(x, rep.a_hat)
        rnorm = float(np.linalg.norm(np.asarray(y, np.float64) - pred))
        d = dict(
            a_hat=rep.a_hat, residual=rep.residual,
            history=np.asarray(rep.residual_norm_history if rep.residual_norm_history is not None else [], np.float64),
            has_history=np.array(rep.residual_norm_history is not None),
            sweeps_run=np.array(rep.sweeps_run), converged=np.array(rep.converged),
            drift_warning=np.array(rep.drift_warning), resid_norm_f64=np.array(rnorm),
            ynorm_f64=np.array(float(np.linalg.norm(np.asarray(y, np.float64)))),
            max_iter=np.array(cfg.max_iter), tol=np.array(cfg.tol),
            ordering=np.array(cfg.ordering), ordering_seed=np.array(cfg.ordering_seed),
            record_history=np.array(cfg.record_history),
            input_sha=np.array(_sha(np.asfortranarray(x), y)),
            dtype=np.array(np.dtype(x.dtype).name),
            shape=np.array(x.shape),
            host=np.array(json.dumps(host)),
            spec=np.array(json.dumps(spec) if spec else ""),
        )
        if a0 is not None:
            d["a0"] = np.asarray(a0)
        if store_inputs:
            d["x"] = np.asfortranarray(x)
            d["y"] = np.asarray(y)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        cases.append(name)
        print(f"{name:28s} {str(x.shape):>16s} {x.dtype} sweeps={rep.sweeps_run} "
              f"conv={rep.converged} |r|={rnorm:.6e}")

    SC = bk.SolveConfig

    # --- known-answer tests of the reference suite (test_solver_bak.py) ---
    add("kat_identity3", np.eye(3, order="F"), np.array([1.0, 2.0, 3.0]), SC(max_iter=1, tol=0))
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((60, 8)))
    xo = np.asfortranarray(q * rng.uniform(0.5, 2.0, 8))
    add("orthogonal_60x8", xo, rng.standard_normal(60), SC(max_iter=1, tol=0))
    rng = np.random.default_rng(14)
    xz = np.asfortranarray(rng.standard_normal((50, 4)))
    xz[:, 2] = 0.0
    yz = rng.standard_normal(50)
    add("zero_column_50x4", xz, yz, SC(max_iter=200, tol=0))
    add("zero_column_warm_50x4", xz, yz, SC(max_iter=50, tol=0), a0=np.array([0.0, 0.0, 7.5, 0.0]))
    add("zero_target_4", np.eye(4, order="F"), np.zeros(4), SC(record_history=True))

    # --- generated systems (pins generate_system too: spec + sha) ---
    def gen(name, obs, nv, seed, prec, cfg, dist="normal", cdist="uniform", sigma=0.01, store=False):
        spec = dict(obs=obs, vars=nv, seed=seed, distribution=dist,
                    coeff_distribution=cdist, noise_sigma=sigma, precision=prec)
        x, y, _ = bk.generate_system(bk.SystemSpec(obs=obs, vars=nv, seed=seed, distribution=dist,
                                                   coeff_distribution=cdist, noise_sigma=sigma), prec)
        add(name, x, y, cfg, spec=spec, store_inputs=store)

    gen("c1_scaled_2000x40_f64", 2000, 40, 1, "double", SC(max_iter=100, tol=0, record_history=True))
    gen("c1_full_10000x100_f64", 10_000, 100, 1, "double", SC(max_iter=100, tol=0, record_history=True))
    gen("c1_scaled_2000x40_f32", 2000, 40, 1, "single", SC(max_iter=100, tol=0, record_history=True))
    gen("early_break_1000x100_f32", 1000, 100, 5, "single", SC(max_iter=300, tol=1e-6, record_history=True),
        dist="uniform", sigma=0.0)
    gen("early_break_400x50_f64", 400, 50, 7, "double", SC(max_iter=5000, tol=1e-12, record_history=True),
        dist="uniform", sigma=0.0)
    gen("random_order_300x30_f64", 300, 30, 9, "double",
        SC(max_iter=40, tol=1e-9, ordering="random", ordering_seed=11, record_history=True))
    gen("random_order_300x30_f32", 300, 30, 9, "single",
        SC(max_iter=40, tol=0, ordering="random", ordering_seed=12, record_history=True))
    gen("c3_scaled_65536x64_f64", 65536, 64, 3, "double", SC(max_iter=5, tol=0, record_history=True))
    gen("c3_scaled_65536x64_f32", 65536, 64, 3, "single", SC(max_iter=5, tol=0, record_history=True))
    for s in range(4):
        gen(f"c5_system{s}_512x32_f32", 512, 32, 5_000_000 + s, "single", SC(max_iter=200, tol=0))

    # --- wide / square / ragged / degenerate, explicit inputs ---
    rng = np.random.default_rng(1001)
    xw = np.asfortranarray(rng.standard_normal((40, 100)))
    add("wide_40x100_f64", xw, xw @ rng.standard_normal(100), SC(max_iter=50, tol=1e-6, record_history=True))
    rng = np.random.default_rng(1002)
    xs = np.asfortranarray(rng.standard_normal((80, 80)).astype(np.float32))
    ys = (xs @ rng.standard_normal(80).astype(np.float32) + 0.5 * rng.standard_normal(80)).astype(np.float32)
    add("square_noisy_80x80_f32", xs, ys,
        SC(max_iter=50, tol=1e-6, ordering="random", ordering_seed=3, record_history=True))
    rng = np.random.default_rng(10)
    xr = np.asfortranarray(rng.standard_normal((37, 9)).astype(np.float32))
    add("ragged_37x9_f32", xr, rng.standard_normal(37).astype(np.float32), SC(max_iter=60, tol=0, record_history=True))
    rng = np.random.default_rng(8)
    x8 = np.asfortranarray(rng.standard_normal((120, 20)).astype(np.float32))
    y8 = (x8 @ rng.standard_normal(20).astype(np.float32) + 0.2 * rng.standard_normal(120)).astype(np.float32)
    add("stagnation_120x20_f32", x8, y8, SC(max_iter=800, tol=0, record_history=True))
    rng = np.random.default_rng(21)
    x1 = np.asfortranarray(rng.standard_normal((33, 1)))
    add("single_column_33x1_f64", x1, rng.standard_normal(33), SC(max_iter=3, tol=0, record_history=True))
    rng = np.random.default_rng(22)
    xc2 = rng.standard_normal(256 * 256).reshape((256, 256), order="F") / 16.0
    xc2[np.arange(256), np.arange(256)] += 4.0
    yc2 = xc2 @ (rng.random(256) * 2 - 1)
    add("c2_scaled_256_f64", xc2, yc2, SC(max_iter=50, tol=0, record_history=True))
    add("c2_scaled_256_f64_break", xc2, yc2, SC(max_iter=50, tol=1e-10, record_history=True))
    rng = np.random.default_rng(23)
    xc4 = np.asfortranarray(rng.standard_normal((100, 3000)))
    add("c4_scaled_100x3000_f64", xc4, rng.standard_normal(100), SC(max_iter=10, tol=0, record_history=True))

    # coordinate_update KAT (test_solver_bak.py:17-20)
    da, e_next = bk.coordinate_update(np.array([1.0, 2.0]), np.array([3.0, 4.0]))
    np.savez_compressed(os.path.join(HERE, "kat_coordinate_update.npz"),
                        col=np.array([1.0, 2.0]), e=np.array([3.0, 4.0]), da=np.array(da), e_next=e_next)
    bakp_cases = make_bakp(bk, host, _predict_f64)
    select_cases = make_select(bk, host)
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump({"host": host, "cases": cases, "bakp_cases": bakp_cases, "select_cases": select_cases,
                   "reference": "baksolve 0.1.0 (/root/reference/pkg)"}, f, indent=1)


def make_bakp(bk, host, _predict_f64):
    """Fixtures of the blocked solver (bakp.py:132-185), files bakp_*.npz.
    A case whose reference solve raises DivergenceError stores the message."""
    cases = []

    def add(name, x, y, cfg, thr, spec=None, store_inputs=True):
        d = dict(thr=np.array(thr), max_iter=np.array(cfg.max_iter), tol=np.array(cfg.tol),
                 record_history=np.array(cfg.record_history), dtype=np.array(np.dtype(x.dtype).name),
                 shape=np.array(x.shape), host=np.array(json.dumps(host)),
                 spec=np.array(json.dumps(spec) if spec else ""),
                 input_sha=np.array(_sha(np.asfortranarray(x), y)))
        try:
            with np.errstate(invalid="ignore", over="ignore"):
                rep = bk.solve_bakp(x, y, bk.BlockConfig(base=cfg, thr=thr, worker_count=1))
        except bk.DivergenceError as err:
            d.update(diverged=np.array(True), message=np.array(str(err)))
            info = f"DivergenceError: {err}"
        else:
            pred = _predict_f64(x, rep.a_hat)
            d.update(diverged=np.array(False), a_hat=rep.a_hat, residual=rep.residual,
                     history=np.asarray(rep.residual_norm_history or [], np.float64),
                     has_history=np.array(rep.residual_norm_history is not None),
                     sweeps_run=np.array(rep.sweeps_run), converged=np.array(rep.converged),
                     drift_warning=np.array(rep.drift_warning),
                     resid_norm_f64=np.array(float(np.linalg.norm(np.asarray(y, np.float64) - pred))),
                     ynorm_f64=np.array(float(np.linalg.norm(np.asarray(y, np.float64)))))
            info = f"sweeps={rep.sweeps_run} conv={rep.converged}"
        if store_inputs:
            d["x"] = np.asfortranarray(x)
            d["y"] = np.asarray(y)
        np.savez_compressed(os.path.join(HERE, f"bakp_{name}.npz"), **d)
        cases.append("bakp_" + name)
        print(f"bakp_{name:24s} {str(x.shape):>14s} {x.dtype} thr={thr} {info}")

    SC = bk.SolveConfig

    def consistent(rng, obs, nv, dtype, noise=0.0):
        x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
        y = (x @ rng.uniform(-1, 1, nv).astype(dtype)).astype(dtype)
        if noise:
            y = (y + noise * rng.standard_normal(obs)).astype(dtype)
        return x, y

    rng = np.random.default_rng(2)
    x, y = consistent(rng, 120, 17, np.float64, 0.1)
    add("thr1_120x17_f64", x, y, SC(max_iter=30, tol=1e-7, record_history=True), 1)
    x, y = consistent(rng, 90, 8, np.float32, 0.1)
    add("thr1_90x8_f32", x, y, SC(max_iter=30, tol=1e-7, record_history=True), 1)
    rng = np.random.default_rng(3)
    x, y = consistent(rng, 250, 48, np.float32, 0.05)
    add("thr16_250x48_f32", x, y, SC(max_iter=25, tol=1e-6, record_history=True), 16)
    rng = np.random.default_rng(6)
    x = np.asfortranarray(rng.standard_normal((35, 10)))
    add("thr4_35x10_f64", x, rng.standard_normal(35), SC(max_iter=3, tol=0, record_history=True), 4)
    rng = np.random.default_rng(5)
    x = np.asfortranarray(rng.standard_normal((40, 7)))
    add("thr3_remainder_40x7_f64", x, x @ np.ones(7), SC(max_iter=1, tol=0), 3)
    rng = np.random.default_rng(4)
    q, _ = np.linalg.qr(rng.standard_normal((60, 8)))
    add("orthonormal_full_60x8_f64", np.asfortranarray(q), rng.standard_normal(60), SC(max_iter=1, tol=0), 8)
    rng = np.random.default_rng(200)
    x, y = consistent(rng, 300, 100, np.float64)
    add("thr10_300x100_f64", x, y, SC(max_iter=60, tol=1e-8, record_history=True), 10)
    rng = np.random.default_rng(31)
    x, y = consistent(rng, 400, 60, np.float32, 0.1)
    add("thr6_400x60_f32", x, y, SC(max_iter=600, tol=0), 6)
    rng = np.random.default_rng(41)
    x = np.asfortranarray(rng.standard_normal((50, 8)))
    x[:, 2] = 0.0
    x[:, 5] = 0.0
    add("zero_columns_50x8_f64", x, rng.standard_normal(50), SC(max_iter=40, tol=0, record_history=True), 4)
    rng = np.random.default_rng(42)
    x = np.asfortranarray(rng.standard_normal((2000, 40)))
    add("thr7_2000x40_f64", x, rng.standard_normal(2000), SC(max_iter=50, tol=0, record_history=True), 7)
    rng = np.random.default_rng(43)
    x = np.asfortranarray(rng.standard_normal((40, 100)))
    add("wide_thr10_40x100_f64", x, x @ rng.standard_normal(100), SC(max_iter=50, tol=1e-6, record_history=True), 10)
    rng = np.random.default_rng(21)
    col = rng.standard_normal(50)
    add("diverge_dup_50x5_f64", np.asfortranarray(np.tile(col[:, None], (1, 5))), col.copy(), SC(max_iter=10), 5)
    add("diverge_nan_2x1_f32", np.asfortranarray(np.array([[1e30], [0.0]], dtype=np.float32)),
        np.array([1e30, 0.0], dtype=np.float32), SC(max_iter=5), 1)
    spec = dict(obs=10000, vars=1000, seed=6, distribution="uniform", coeff_distribution="uniform",
                noise_sigma=0.0, precision="single")
    x, y, _ = bk.generate_system(bk.SystemSpec(obs=10000, vars=1000, seed=6), "single")
    add("paper_10000x1000_f32_thr50", x, y, SC(max_iter=200, tol=1e-6, record_history=True), 50, spec=spec,
        store_inputs=False)
    # block_deltas KATs (test_solver_bakp.py:18-34)
    np.savez_compressed(os.path.join(HERE, "kat_block_deltas.npz"),
                        eye=bk.block_deltas(np.eye(2, order="F"), (0, 2), np.array([3.0, 4.0])),
                        dup=bk.block_deltas(np.asfortranarray(np.column_stack([[1.0, 2.0, -1.0]] * 2)), (0, 2),
                                            np.array([1.0, 2.0, -1.0])))
    return cases



def make_select(bk, host):
    """Fixtures of score_all_columns / select_features (select.py:56-136),
    files select_*.npz: inputs plus the reference's outputs."""
    cases = []

    def randn(rng, obs, nv, dtype=np.float64):
        return np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))

    def score(name, x, e, excluded=()):
        try:
            best, scores = bk.score_all_columns(x, e, excluded=list(excluded))
            d = dict(best=np.array(best), scores=scores, exhausted=np.array(False))
        except bk.SelectionExhaustedError:
            d = dict(best=np.array(-1), scores=np.zeros(0), exhausted=np.array(True))
        np.savez_compressed(os.path.join(HERE, f"select_{name}.npz"), kind=np.array("score"), x=x, e=e,
                            excluded=np.asarray(sorted(excluded), dtype=np.int64), host=np.array(json.dumps(host)),
                            **d)
        cases.append("select_" + name)
        print(f"select_{name:30s} score best={int(d['best'])}")

    def select(name, x, y, max_feat, refit="qr", stop_tol=0.0, refit_cfg=None):
        cfg = bk.FeatureSelectConfig(max_feat=max_feat, refit=refit, stop_tol=stop_tol,
                                     refit_config=bk.SolveConfig(**refit_cfg) if refit_cfg else None)
        rep = bk.select_features(x, y, cfg)
        np.savez_compressed(os.path.join(HERE, f"select_{name}.npz"), kind=np.array("select"), x=x, y=y,
                            max_feat=np.array(max_feat), refit=np.array(refit), stop_tol=np.array(stop_tol),
                            refit_cfg=np.array(json.dumps(refit_cfg or {})),
                            selected=np.asarray(rep.selected, dtype=np.int64),
                            residual_norms=np.asarray(rep.residual_norms, dtype=np.float64),
                            final_coeffs=np.asarray(rep.final_coeffs), host=np.array(json.dumps(host)))
        cases.append("select_" + name)
        print(f"select_{name:30s} selected={rep.selected}")

    rng = np.random.default_rng(40)
    x = randn(rng, 30, 6)
    score("explains_30x6", x, x[:, 3].copy())
    rng = np.random.default_rng(42)
    score("random_20x5", randn(rng, 20, 5), rng.standard_normal(20))
    rng = np.random.default_rng(43)
    score("f32_400x30", randn(rng, 400, 30, np.float32), rng.standard_normal(400).astype(np.float32))
    rng = np.random.default_rng(44)
    x = randn(rng, 30, 4)
    x[:, 2] = 0.0
    e = x[:, 1].copy()
    score("zero_col_excluded_30x4", x, e, excluded=[1])
    score("exhausted_30x4", x, e, excluded=[0, 1, 3])
    rng = np.random.default_rng(56)
    col = rng.standard_normal(25)
    score("tie_25x3", np.asfortranarray(np.column_stack([col, col, col])), rng.standard_normal(25))
    rng = np.random.default_rng(60)
    score("tall_16384x16", randn(rng, 16384, 16), rng.standard_normal(16384))
    rng = np.random.default_rng(61)
    score("wide_100x2000_f32", randn(rng, 100, 2000, np.float32), rng.standard_normal(100).astype(np.float32))

    def sparse(rng, obs, nv, k):
        x = randn(rng, obs, nv)
        sup = sorted(rng.choice(nv, size=k, replace=False).tolist())
        a = np.zeros(nv)
        a[sup] = rng.uniform(1.0, 2.0, k) * rng.choice([-1.0, 1.0], k)
        return x, x @ a

    for seed in (3000, 3001):
        x, y = sparse(np.random.default_rng(seed), 500, 50, 3)
        select(f"support_{seed}_500x50", x, y, 3)
    rng = np.random.default_rng(46)
    x = randn(rng, 60, 8)
    select("full_60x8", x, rng.standard_normal(60), 8)
    x, y = sparse(np.random.default_rng(47), 200, 30, 2)
    select("stop_tol_200x30", x, y, 10, stop_tol=1e-8)
    x, y = sparse(np.random.default_rng(48), 300, 40, 4)
    select("bak_refit_300x40", x, y, 4, refit="bak", refit_cfg=dict(max_iter=4000, tol=1e-10))
    rng = np.random.default_rng(49)
    x = randn(rng, 80, 10)
    x[:, 4] = 0.0
    select("zero_col_80x10", x, rng.standard_normal(80), 9)
    rng = np.random.default_rng(62)
    x = randn(rng, 2000, 100, np.float32)
    y = (x[:, [3, 17, 60]] @ np.array([1.5, -2.0, 0.7], np.float32) + 0.01 * rng.standard_normal(2000)).astype(
        np.float32)
    select("f32_bak_2000x100", x, y, 5, refit="bak", refit_cfg=dict(max_iter=200, tol=1e-7))
    return cases


def make_matio(bk):
    """Files written by the reference's save_matrix (matio.py:29-39): a
    binary f64, a binary f32 and a CSV, plus the matrices they hold."""
    rng = np.random.default_rng(65)
    x64 = np.asfortranarray(rng.standard_normal((13, 4)))
    x64[0, 0], x64[1, 1], x64[2, 2] = 1.0 / 3.0, 1e-300, -1e308
    x32 = np.asfortranarray(rng.standard_normal((7, 3)).astype(np.float32))
    bk.save_matrix(os.path.join(HERE, "matio_f64.bakm"), x64, format="binary")
    bk.save_matrix(os.path.join(HERE, "matio_f32.bakm"), x32, format="binary")
    bk.save_matrix(os.path.join(HERE, "matio_f64.csv"), x64, format="csv")
    np.savez_compressed(os.path.join(HERE, "matio_expected.npz"), x64=x64, x32=x32)
    print("matio fixtures written")


def make_harness(bk):
    """Records of the reference's run_case (bench.py:137-195) for a few small
    generated cases (wall time dropped): the harness's metrics must agree."""
    import dataclasses
    cases = [
        dict(case_id="s400_bak", solver="bak", obs=400, vars=40, seed=7, precision="single", tol=1e-6,
             max_iter=300),
        dict(case_id="s400_bakp", solver="bakp", obs=400, vars=40, seed=7, precision="single", tol=1e-6,
             max_iter=300, thr=8),
        dict(case_id="s400_qr", solver="qr", obs=400, vars=40, seed=7, precision="single", tol=1e-6,
             max_iter=300),
        dict(case_id="d1000_bak", solver="bak", obs=1000, vars=100, seed=5, precision="double", tol=1e-10,
             max_iter=2000),
        dict(case_id="d1000_coeffs", solver="qr", obs=1000, vars=100, seed=5, precision="double", tol=1e-6,
             max_iter=300, mape_base="coeffs"),
        dict(case_id="p2000_bakp", solver="bakp", obs=2000, vars=200, seed=11, precision="single", tol=1e-6,
             max_iter=200, thr=20),
    ]
    out = []
    for c in cases:
        spec = bk.RunSpec(case_id=c["case_id"], solver=c["solver"],
                          system=bk.SystemSpec(obs=c["obs"], vars=c["vars"], seed=c["seed"]),
                          precision=c["precision"], thr=c.get("thr", 50), tol=c["tol"], max_iter=c["max_iter"],
                          repetitions=1, mape_base=c.get("mape_base", "targets"))
        rec = dataclasses.asdict(bk.run_case(spec))
        rec.pop("wall_time_s")
        out.append(dict(spec=c, record=rec))
        print(c["case_id"], rec["sweeps"], rec["mape"], rec["rel_residual"])
    with open(os.path.join(HERE, "harness_records.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
