"""B200 artifact runner: the `triton_runner` contract on the native backend.

Drop-in for `python -m triton_runner run` (reference
pkg/triton_runner/src/triton_runner/cli.py:25-83, runner.py:62-210): the same
inputs - a manifest sidecar written by `tiledsl emit` (emit.py:296-308),
TWT1 / JSON tensor files written by `tiledsl simulate --save-dir`
(tensorio.py:18-69), `--meta NAME=INT` values - the same validation errors,
the same max-abs comparison and the same exit codes:

    0 pass   1 mismatch   2 usage / artifact error   3 no GPU / backend

The difference is the executor: the manifest's kernel name selects this
package's catalog spec (which is tree-identical to the reference's), checked
against the manifest's parameter list, and the kernel runs through
`backend.launch` on the sm_100a library.  `--source` (the emitted Triton
file) is accepted for command-line compatibility and only checked to exist
when given.  Rank-0 parameters (addmm beta/alpha, stored as rank-0 TWT1
files) are passed by value, which is what the kernel ABI wants (emit.py:84-85).

    python -m paper_2507_11978_b200.runner run --manifest mm/mm.manifest.json \\
        --inputs input=mm/input.twt --inputs other=mm/other.twt \\
        --expect mm/expected.twt --meta BLOCK_SIZE_M=2 --meta BLOCK_SIZE_N=2 --meta BLOCK_SIZE_K=2
"""

from __future__ import annotations

import argparse
import json
import struct
import sys
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

EXIT_OK, EXIT_FAIL, EXIT_USAGE, EXIT_NO_ENV = 0, 1, 2, 3
KINDS = ("f16", "f32")
ROLES = ("in", "out")
TWT_MAGIC = b"TWT1"


class ManifestError(Exception):
    """Manifest or artifact set is missing, malformed or inconsistent."""


class TensorIOError(Exception):
    """Tensor file missing, truncated or malformed."""


class EnvironmentUnavailable(Exception):
    """No CUDA device / native library."""


# ---- tensor files (TWT1: magic, u32 rank, u32 sizes, f32 LE payload) --------

def read_tensor(path) -> np.ndarray:
    path = Path(path)
    try:
        raw = path.read_bytes()
    except OSError as exc:
        raise TensorIOError(f"cannot read {path}: {exc}") from exc
    if path.suffix == ".json":
        try:
            doc = json.loads(raw)
            shape = tuple(int(s) for s in doc["shape"])
            return np.asarray(doc["data"], dtype=np.float32).reshape(shape)
        except (ValueError, KeyError, TypeError) as exc:
            raise TensorIOError(f"{path}: malformed JSON tensor: {exc}") from exc
    if len(raw) < 8 or raw[:4] != TWT_MAGIC:
        raise TensorIOError(f"{path}: not a TWT1 tensor file")
    rank = struct.unpack_from("<I", raw, 4)[0]
    head = 8 + 4 * rank
    if len(raw) < head:
        raise TensorIOError(f"{path}: truncated header")
    shape = struct.unpack_from(f"<{rank}I", raw, 8)
    count = int(np.prod(shape)) if rank else 1
    if len(raw) != head + 4 * count:
        raise TensorIOError(f"{path}: expected {head + 4 * count} bytes for shape "
                            f"{tuple(shape)}, got {len(raw)}")
    return np.frombuffer(raw, dtype="<f4", offset=head, count=count).reshape(shape).astype(np.float32)


def write_tensor(path, arr) -> None:
    arr = np.ascontiguousarray(arr, dtype="<f4")
    with open(path, "wb") as f:
        f.write(TWT_MAGIC + struct.pack("<I", arr.ndim) + struct.pack(f"<{arr.ndim}I", *arr.shape))
        f.write(arr.tobytes())


# ---- manifest --------------------------------------------------------------

@dataclass(frozen=True)
class Param:
    name: str
    rank: int
    kind: str
    role: str


@dataclass(frozen=True)
class Manifest:
    name: str
    params: tuple
    meta: tuple
    launcher_args: tuple


def _manifest_problems(m: Manifest) -> list:
    """Everything wrong with a parsed manifest, so one error reports all."""
    problems = []
    for p in m.params:
        if p.kind not in KINDS:
            problems.append(f"{p.name}: element kind {p.kind!r} is not one of {'/'.join(KINDS)}")
        if p.role not in ROLES:
            problems.append(f"{p.name}: role {p.role!r} is neither 'in' nor 'out'")
        if p.rank < 0:
            problems.append(f"{p.name}: rank {p.rank} < 0")
    order = tuple(p.name for p in m.params) + m.meta
    if m.launcher_args != order:
        problems.append(f"launcher argument order {list(m.launcher_args)} is not parameters "
                        f"then meta {list(order)}")
    n_out = sum(p.role == "out" for p in m.params)
    if n_out != 1:
        problems.append(f"{n_out} output parameters; the runner compares exactly one")
    return problems


def load_manifest(path) -> Manifest:
    """Parse and validate the sidecar that `tiledsl emit` writes next to a
    kernel (the reference's emit.py:296-308 schema)."""
    path = Path(path)
    try:
        doc = json.loads(path.read_bytes())
        if not isinstance(doc, dict):
            raise TypeError("top level is not an object")
        m = Manifest(
            name=str(doc["name"]),
            params=tuple(Param(str(e["name"]), int(e["rank"]), str(e["kind"]), str(e["role"]))
                         for e in doc["params"]),
            meta=tuple(map(str, doc["meta"])),
            launcher_args=tuple(map(str, doc["launcher_args"])))
    except OSError as exc:
        raise ManifestError(f"manifest {path} unreadable: {exc}") from exc
    except (ValueError, KeyError, TypeError) as exc:
        raise ManifestError(f"manifest {path} is not a kernel manifest ({exc})") from exc
    problems = _manifest_problems(m)
    if problems:
        raise ManifestError(f"manifest {path}: " + "; ".join(problems))
    return m


def default_tolerance(m: Manifest) -> float:
    return 1e-2 if any(p.kind == "f16" for p in m.params) else 1e-4


@dataclass
class Request:
    manifest: Manifest
    inputs: dict
    expected: np.ndarray
    meta: dict
    tol: float


@dataclass
class Report:
    kernel: str
    max_abs: float
    tol: float
    passed: bool
    details: dict = field(default_factory=dict)


def _as_param_array(arr: np.ndarray, p: Param) -> np.ndarray:
    # `tiledsl simulate --save-dir` writes rank-0 scalars (addmm beta / alpha)
    # through np.ascontiguousarray, i.e. with shape (1,) (tensorio.py:25-36,
    # cli.py:217-222): a one-element file feeds a rank-0 parameter
    return arr.reshape(()) if p.rank == 0 and arr.size == 1 else arr


def build_request(manifest_path, input_paths: dict, expect_path, meta: dict, tol=None,
                  source=None) -> Request:
    """Load every artifact and check it against the manifest; all problems
    with names (inputs, meta) are reported together."""
    if source is not None and not Path(source).is_file():
        raise ManifestError(f"--source {source} does not exist")
    m = load_manifest(manifest_path)
    ins = {p.name: p for p in m.params if p.role == "in"}
    problems = [f"no tensor file for input {n!r}" for n in sorted(set(ins) - set(input_paths))]
    problems += [f"{n!r} is not an input of {m.name}" for n in sorted(set(input_paths) - set(ins))]
    problems += [f"no value for meta {n}" for n in sorted(set(m.meta) - set(meta))]
    problems += [f"{n} is not a meta-parameter of {m.name}" for n in sorted(set(meta) - set(m.meta))]
    problems += [f"meta {n}={v} is not positive" for n, v in sorted(meta.items()) if v <= 0]
    if problems:
        raise ManifestError("; ".join(problems))
    inputs = {n: _as_param_array(read_tensor(path), ins[n]) for n, path in input_paths.items()}
    wrong = [f"{n}: {path} holds a rank-{inputs[n].ndim} tensor, {m.name} takes rank "
             f"{ins[n].rank}" for n, path in input_paths.items() if inputs[n].ndim != ins[n].rank]
    expected = read_tensor(expect_path)
    out = next(p for p in m.params if p.role == "out")
    if expected.ndim != out.rank:
        wrong.append(f"expected output {expect_path} is rank {expected.ndim}, {out.name} is rank "
                     f"{out.rank}")
    if wrong:
        raise ManifestError("; ".join(wrong))
    return Request(m, inputs, expected, dict(meta),
                   default_tolerance(m) if tol is None else float(tol))


def run_and_compare(req: Request) -> Report:
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise EnvironmentUnavailable(f"torch not importable: {exc}") from exc
    if not torch.cuda.is_available():
        raise EnvironmentUnavailable("no CUDA device available")
    from . import backend
    from .catalog import ALL_NAMES, checked

    m = req.manifest
    if m.name not in ALL_NAMES:
        raise ManifestError(f"no B200 kernel for manifest {m.name!r}")
    ck = checked(m.name)
    if [(p.name, p.rank, p.role) for p in ck.spec.params] != \
            [(p.name, p.rank, p.role) for p in m.params]:
        raise ManifestError(f"manifest parameters do not match the {m.name} kernel")
    dtypes = {"f16": torch.float16, "f32": torch.float32}
    args = {}
    for p in m.params:
        if p.rank == 0 and p.role == "in":
            args[p.name] = float(np.asarray(req.inputs[p.name]).reshape(()))
        elif p.role == "out":
            args[p.name] = torch.zeros(req.expected.shape, device="cuda", dtype=dtypes[p.kind])
        else:
            args[p.name] = torch.from_numpy(req.inputs[p.name]).to("cuda", dtypes[p.kind])
    try:
        backend.launch(ck, args, req.meta)
        torch.cuda.synchronize()
    except backend.LaunchError as exc:
        raise ManifestError(f"launch rejected: {exc}") from exc
    except (backend.BackendError, RuntimeError) as exc:
        raise EnvironmentUnavailable(f"B200 backend failure: {exc}") from exc
    out = next(p for p in m.params if p.role == "out")
    got = args[out.name].float().cpu().numpy()
    max_abs = float(np.max(np.abs(got - req.expected))) if got.size else 0.0
    return Report(m.name, max_abs, req.tol, max_abs <= req.tol,
                  {"output_shape": list(got.shape), "paths": backend.path_counts()})


def _pairs(items, label, conv):
    out = {}
    for item in items:
        name, sep, value = item.partition("=")
        if not sep or not name:
            raise ManifestError(f"bad {label} {item!r}, expected NAME=VALUE")
        if name in out:
            raise ManifestError(f"duplicate {label} {name!r}")
        try:
            out[name] = conv(value)
        except ValueError as exc:
            raise ManifestError(f"bad {label} {item!r}: {exc}") from exc
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="b200-runner",
                                 description="run a manifest's kernel on the B200 backend and "
                                             "compare against an expected tensor")
    sub = ap.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run")
    r.add_argument("--source", default=None, help="emitted kernel file (accepted, not executed)")
    r.add_argument("--manifest", required=True)
    r.add_argument("--inputs", action="append", default=[], metavar="NAME=PATH")
    r.add_argument("--expect", required=True)
    r.add_argument("--meta", action="append", default=[], metavar="NAME=INT")
    r.add_argument("--tol", type=float, default=None)
    args = ap.parse_args(argv)
    try:
        req = build_request(args.manifest, _pairs(args.inputs, "input", str), args.expect,
                            _pairs(args.meta, "meta", int), args.tol, args.source)
    except (ManifestError, TensorIOError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    try:
        rep = run_and_compare(req)
    except EnvironmentUnavailable as exc:
        print(f"environment unavailable: {exc}", file=sys.stderr)
        return EXIT_NO_ENV
    except ManifestError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    print(f"{rep.kernel}: max-abs {rep.max_abs:.3e} tol {rep.tol:.0e} "
          f"{'pass' if rep.passed else 'FAIL'}")
    return EXIT_OK if rep.passed else EXIT_FAIL


if __name__ == "__main__":
    sys.exit(main())
