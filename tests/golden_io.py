"""Load the committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the real reference)."""

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("kat_coordinate", "kat_block_deltas", "bakp_", "select_", "matio_",
                                                          "fullsize_")))


def fullsize(name):
    """Full-size reference outputs (make_golden_fullsize.py): dict of arrays."""
    with np.load(os.path.join(GOLDEN, f"fullsize_{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def bakp_names():
    """Fixtures of the blocked solver (bakp.py), made by make_golden.make_bakp."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "bakp_*.npz")))


def load_bakp(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    spec = str(d["spec"])
    if "x" not in d:
        from oracle import bak_oracle as orc
        s = json.loads(spec)
        x, y, _ = orc.make_system(s["obs"], s["vars"], s["seed"], s["distribution"],
                                  s["coeff_distribution"], s["noise_sigma"], s["precision"])
        d["x"], d["y"] = x, y
    d["config"] = dict(max_iter=int(d["max_iter"]), tol=float(d["tol"]), record_history=bool(d["record_history"]))
    d["thr"] = int(d["thr"])
    d["diverged"] = bool(d["diverged"])
    d["host"] = json.loads(str(d["host"]))
    return d


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    spec = str(d["spec"])
    if "x" not in d:
        from oracle import bak_oracle as orc
        s = json.loads(spec)
        x, y, _ = orc.make_system(s["obs"], s["vars"], s["seed"], s["distribution"],
                                  s["coeff_distribution"], s["noise_sigma"], s["precision"])
        d["x"], d["y"] = x, y
    d["config"] = dict(max_iter=int(d["max_iter"]), tol=float(d["tol"]), ordering=str(d["ordering"]),
                       ordering_seed=int(d["ordering_seed"]), record_history=bool(d["record_history"]))
    d["a0"] = d.get("a0")
    d["host"] = json.loads(str(d["host"]))
    return d


def input_sha(x, y):
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(np.asfortranarray(x)).tobytes())
    h.update(np.ascontiguousarray(y).tobytes())
    return h.hexdigest()


def select_names(kind=None):
    """Fixtures of score_all_columns / select_features (make_golden.make_select)."""
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "select_*.npz"))):
        name = os.path.basename(p)[:-4]
        if kind is None or str(np.load(p)["kind"]) == kind:
            out.append(name)
    return out


def load_select(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    d["kind"] = str(d["kind"])
    d["host"] = json.loads(str(d["host"]))
    if d["kind"] == "select":
        d["refit"] = str(d["refit"])
        d["refit_cfg"] = json.loads(str(d["refit_cfg"]))
        d["max_feat"] = int(d["max_feat"])
        d["stop_tol"] = float(d["stop_tol"])
        d["selected"] = d["selected"].tolist()
    else:
        d["excluded"] = d["excluded"].tolist()
        d["best"] = int(d["best"])
        d["exhausted"] = bool(d["exhausted"])
    return d
