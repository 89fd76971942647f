"""Loader for the committed golden fixtures (tests/golden/*.npz, made by make_golden.py)."""
import ast
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pipeline_cases():
    z = np.load(os.path.join(HERE, "pipeline_cases.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("__", 1)
        cases.setdefault(name, {})[field] = z[key]
    for c in cases.values():
        c["params"] = ast.literal_eval(str(c["params"]))
    return cases


def stage_cases():
    z = np.load(os.path.join(HERE, "stage_cases.npz"))
    return {k: z[k] for k in z.files}


def params_obj(d):
    from oracle.dehaze_oracle import OracleParams

    return OracleParams(**d)
