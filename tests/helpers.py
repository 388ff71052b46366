"""Fixture access shared by the tests (golden vectors from the reference)."""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def maps():
    return json.loads((GOLDEN / "maps.json").read_text())


@lru_cache(maxsize=None)
def map_cases():
    return json.loads((GOLDEN / "map_points.json").read_text()), dict(
        np.load(GOLDEN / "map_points.npz"))


@lru_cache(maxsize=None)
def sim_cases():
    return json.loads((GOLDEN / "sim_cases.json").read_text()), dict(
        np.load(GOLDEN / "sim_cases.npz"))


@lru_cache(maxsize=None)
def expr_cases():
    return json.loads((GOLDEN / "expr_cases.json").read_text())


def case_args(ci, case, arrays):
    """Reference launch arguments of one sim case (inputs + scalars)."""
    args = {n: arrays[f"c{ci}_{n}"] for n in case["inputs"]}
    args.update(case["scalars"])
    return args


def run_oracle(kernel, args, meta):
    import oracle

    if kernel == "add":
        return oracle.add(args["input"], args["other"])
    if kernel == "silu":
        return oracle.silu(args["input"])
    if kernel == "softmax":
        return oracle.softmax(args["input"], meta["COLS_PADDED"])
    if kernel == "rms_norm":
        return oracle.rms_norm(args["input"], args["weight"])
    if kernel == "mm":
        return oracle.mm(args["input"], args["other"])
    if kernel == "bmm":
        return oracle.bmm(args["input"], args["other"])
    if kernel == "addmm":
        return oracle.addmm(args["input"], args["mat1"], args["mat2"], args["beta"],
                            args["alpha"])
    if kernel == "conv2d":
        return oracle.conv2d(args["input"], args["filter"])
    raise ValueError(kernel)


def out_shape(kernel, args):
    if kernel in ("add", "silu", "softmax", "rms_norm"):
        return args["input"].shape
    if kernel == "mm":
        return (args["input"].shape[0], args["other"].shape[1])
    if kernel == "bmm":
        return (args["input"].shape[0], args["input"].shape[1], args["other"].shape[2])
    if kernel == "addmm":
        return args["input"].shape
    if kernel == "conv2d":
        n, c, h, w = args["input"].shape
        k, _, r, s = args["filter"].shape
        return (n, k, h - r + 1, w - s + 1)
    raise ValueError(kernel)
