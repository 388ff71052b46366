"""The drop-in B200 executor: ``launch`` (twin of the reference's
``sim.launch``) and the per-kernel ``{name}_launch`` launchers (twins of the
emitted Triton launchers).

Reference contracts mirrored here:

* ``launch(checked, args, meta)`` - sim.py:163-236.  Same argument
  validation and ``LaunchError`` conditions (missing / non-positive /
  unexpected meta, missing / unexpected argument, wrong rank,
  sim.py:128-150), same launch-time checks (sim.py:153-160) and grid
  evaluation (sim.py:176-183, "grid dimension evaluated to g").  ``args``
  maps parameter names to CUDA ``torch.Tensor``s (strides in elements, as
  ``ConcreteTensor.strides``) and rank-0 parameters to Python floats.
  Returns ``LaunchResult(grid, total)``.
* ``{name}_launch(*params, *meta)`` - emit.py:267-293: positional
  parameters in KernelSpec order, then meta; reads ``.shape``/``.stride()``,
  asserts the checks, launches, returns the out-parameters.

Execution: the CheckedSpec's maps are compiled to the native map VM
(bytecode.py) which evaluates checks and grid; the spec is matched to a
kernel family by name AND by structural identity of its grid, checks,
index maps and application IR with this package's catalog (so a spec built
by the reference front end is accepted only if it computes what the native
kernel computes); then ``ntb_launch`` runs the hand-written sm_100a kernel.
Unmatched specs raise ``UnsupportedSpecError``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Mapping, Optional

import numpy as np

from . import _lib
from . import symbolic as se
from .bytecode import MapProgram, build_program
from .catalog import ALL_NAMES, checked as canonical
from .spec import ir_tree


class LaunchError(Exception):
    """Bad launch configuration (reference sim.LaunchError, sim.py:39-41)."""


class UnsupportedSpecError(LaunchError):
    """The spec does not match any sm_100a kernel family."""


class BackendError(RuntimeError):
    """CUDA / native-library failure."""


@dataclass(frozen=True)
class LaunchResult:
    grid: tuple
    total: int
    # collect_writes=True: per out-parameter, per program (forward pid order),
    # the sorted flat offsets the program writes (sim.LaunchResult.writes)
    writes: Optional[dict] = None


_DTYPES = None


def _dtype_code(t):
    global _DTYPES
    import torch

    if _DTYPES is None:
        _DTYPES = {torch.float32: _lib.NTB_F32, torch.float16: _lib.NTB_F16,
                   torch.bfloat16: _lib.NTB_BF16}
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise LaunchError(f"unsupported element type {t.dtype}") from None


# ---- spec -> (family, program) cache --------------------------------------

_cache_lock = threading.Lock()
_cache: dict = {}


def _rename_tree(t, ren):
    """JSON-form expression tree with symbols renamed."""
    if t[0] == "sym":
        return ["sym", ren.get(t[1], t[1])]
    if t[0] == "const":
        return list(t)
    return [t[0]] + [_rename_tree(a, ren) for a in t[1:]]


def _canon_ir(node, ren, params, scope):
    """ir_tree() output with parameters positional and locals / loop
    variables numbered by first appearance (alpha-renaming)."""
    if isinstance(node, list) and node and isinstance(node[0], str) and node[0] == "expr":
        return ["expr", _rename_tree(node[1], ren)]
    if isinstance(node, list) and node and isinstance(node[0], str) and node[0][:1].isupper():
        cls = node[0]
        out = [cls]
        for field, value in node[1:]:
            if field == "param":
                value = params.get(value, value)
            elif field == "name" and cls in ("Let", "Assign", "Accumulate", "Local", "Var"):
                value = scope.setdefault(("l", value), f"l{len(scope)}")
            elif field == "var" and cls == "ForRange":
                value = scope.setdefault(("l", value), f"l{len(scope)}")
            else:
                value = _canon_ir(value, ren, params, scope)
            out.append([field, value])
        return out
    if isinstance(node, list):
        return [_canon_ir(x, ren, params, scope) for x in node]
    return node


def _node(n, *classes):
    return isinstance(n, list) and n and isinstance(n[0], str) and n[0] in classes


def _reads(n, acc):
    """Names of the locals an ir_tree() expression reads."""
    if _node(n, "Local"):
        acc.add(dict(n[1:])["name"])
    if isinstance(n, list):
        for x in n:
            _reads(x, acc)
    return acc


def _writes(n, acc):
    """Names of the locals a statement (or block) Assigns / Accumulates."""
    if _node(n, "Accumulate", "Assign"):
        acc.add(dict(n[1:])["name"])
    if isinstance(n, list):
        for x in n:
            _writes(x, acc)
    return acc


def _inline_lets(stmts):
    """Inline single-assignment locals (a Let whose name is never Accumulate'd
    or Assign'ed) into their uses, on the ir_tree() form, so that equivalent
    formulations of the same application (e.g. the paper's softmax with its
    `row_minus_max` temporaries vs the catalog's) compare equal.

    A Let that reads a MUTABLE local is a snapshot: it is inlined only when
    no write to that local can happen between the Let and any of its uses
    (later in the same block, or anywhere in an enclosing loop body that
    does not also contain the Let).  Otherwise it stays a Let, so a spec that
    reads a frozen copy of a running value never fingerprints like one that
    reads the live value."""
    mutable = _writes(stmts, set())
    defs = {}

    def sub(n):
        if _node(n, "Local"):
            name = dict(n[1:])["name"]
            if name in defs:
                return defs[name]
        if isinstance(n, list):
            return [sub(x) for x in n]
        return n

    def safe(name, deps, rest):
        """rest: the statements after the Let in its block.  (A Let inside a
        loop body re-snapshots every iteration, so only the rest of its own
        block can put a write between it and a use.)"""
        if not deps:
            return True
        written = set()
        for st in rest:
            if written & deps and name in _reads(st, set()):
                return False
            if _node(st, "ForRange"):
                body = dict(st[1:])["body"]
                if _writes(body, set()) & deps and name in _reads(body, set()):
                    return False
            written |= _writes(st, set())
        return True

    def block(ss):
        out = []
        for i, st in enumerate(ss):
            if _node(st, "Let"):
                f = dict(st[1:])
                name = f["name"]
                expr = sub(f["expr"])
                if name not in mutable and safe(name, _reads(expr, set()) & mutable, ss[i + 1:]):
                    defs[name] = expr
                    continue
                defs.pop(name, None)
                out.append([st[0]] + [[k, expr if k == "expr" else v] for k, v in st[1:]])
                continue
            if _node(st, "ForRange"):
                st = [st[0]] + [[k, block(v) if k == "body" else sub(v)] for k, v in st[1:]]
                out.append(st)
                continue
            out.append(sub(st))
        return out

    return block(stmts)


def _fingerprint(checked):
    """Identity of a CheckedSpec - grid, checks, maps, IR - with parameter,
    meta, local and kernel names factored out, so that any spec that
    computes the same thing (e.g. one written through make()) matches.
    Integer maps are compared by their canonical form (symbolic.canonical:
    polynomial normal form over floor-div / mod atoms), so the front end
    that built them - this package's, the reference's, a user's - and the
    order it built them in do not matter; launch checks are compared as an
    orientation-free set."""
    spec = checked.spec
    ren, params = {}, {}
    for i, p in enumerate(spec.params):
        params[p.name] = f"p{i}"
        for d in range(p.rank):
            ren[f"{p.name}_size_{d}"] = f"p{i}_size_{d}"
            ren[f"{p.name}_stride_{d}"] = f"p{i}_stride_{d}"
    for j, m in enumerate(spec.meta):
        ren[m] = f"m{j}"

    def tr(e):
        return se.canonical(se.from_tree(_rename_tree(se.to_tree(se.from_any(e)), ren)))

    maps = []
    for p in spec.params:
        if p.rank < 1:
            continue
        m = checked.index_maps[p.name]
        maps.append((
            params[p.name],
            tuple(tr(s) for s in m.lane_sizes),
            tuple(tr(s) for s in m.nest_sizes),
            tr(m.offset),
            tuple((tr(a), tr(b)) for a, b in m.mask),
        ))
    return (
        tuple((p.rank, p.role) for p in spec.params),
        len(spec.meta),
        tuple(tr(s) for s in checked.grid.sizes),
        frozenset(frozenset((tr(a), tr(b))) for a, b in checked.grid.checks),
        tuple(maps),
        repr(_canon_ir(_inline_lets(ir_tree(spec.application)), ren, params, {})),
    )


_canon_fps: dict = {}


def _family_of(checked) -> str:
    fp = _fingerprint(checked)
    name = checked.spec.name
    if name in ALL_NAMES:
        if name not in _canon_fps:
            _canon_fps[name] = _fingerprint(canonical(name))
        if _canon_fps[name] == fp:
            return name
    for fam in ALL_NAMES:
        if fam not in _canon_fps:
            _canon_fps[fam] = _fingerprint(canonical(fam))
        if _canon_fps[fam] == fp:
            return fam
    raise UnsupportedSpecError(
        f"spec {name!r} does not match any sm_100a kernel family (add, silu, softmax, rms_norm, "
        "mm, bmm, addmm, conv2d, sdpa, rope); the B200 backend executes only specs whose "
        "arrangement and application it has a native kernel for")


def _resolve(checked, allow_generic: bool = False) -> tuple:
    """(family, map program).  family is None for a spec that matches no
    native kernel family when ``allow_generic`` (the generated-code path)."""
    key = id(checked)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0] is checked:
            if hit[1] is None and not allow_generic:
                _family_of(checked)   # raises UnsupportedSpecError
            return hit[1], hit[2]
    try:
        family = _family_of(checked)
    except UnsupportedSpecError:
        if not allow_generic:
            raise
        family = None
    prog = build_program(checked)
    with _cache_lock:
        _cache[key] = (checked, family, prog)
    return family, prog


# ---- binding and validation (sim.py:120-160) ------------------------------

def _binding(spec, args: Mapping, meta: Mapping) -> dict:
    binding: dict = {}
    for name in spec.meta:
        if name not in meta:
            raise LaunchError(f"missing meta-parameter {name!r}")
        v = int(meta[name])
        if v < 1:
            raise LaunchError(f"meta-parameter {name!r} must be positive, got {v}")
        binding[name] = v
    for extra in sorted(set(meta) - set(spec.meta)):
        raise LaunchError(f"unexpected meta-parameter {extra!r}")
    for p in spec.params:
        if p.name not in args:
            raise LaunchError(f"missing argument {p.name!r}")
        t = args[p.name]
        if p.rank == 0:
            continue
        shape = tuple(t.shape)
        if len(shape) != p.rank:
            raise LaunchError(f"argument {p.name!r} has rank {len(shape)}, expected {p.rank}")
        for i, (size, stride) in enumerate(zip(shape, t.stride())):
            binding[f"{p.name}_size_{i}"] = int(size)
            binding[f"{p.name}_stride_{i}"] = int(stride)
    for extra in sorted(set(args) - {p.name for p in spec.params}):
        raise LaunchError(f"unexpected argument {extra!r}")
    return binding


def _check_failure(prog: MapProgram, binding: dict) -> str:
    for (lt, rt), (lhs, rhs) in zip(prog.checks_text, prog.grid.checks):
        lv, rv = se.evaluate(lhs, binding), se.evaluate(rhs, binding)
        if lv != rv:
            return f"launch-time check failed: {lt} = {lv} but {rt} = {rv}"
    return _lib.last_error()


def evaluate_grid(checked, binding: dict) -> tuple:
    """Checks + grid through the native map VM (ntb_grid_eval)."""
    _, prog = _resolve(checked, allow_generic=True)
    rc, grid = _lib.grid_eval(prog.blob, prog.slots(binding))
    if rc == _lib.NTB_ERR_CHECK:
        raise LaunchError(_check_failure(prog, binding))
    if rc == _lib.NTB_ERR_EVAL:
        raise LaunchError(_lib.last_error())
    if rc:
        raise BackendError(_lib.last_error())
    return grid


_plans: dict = {}
_PLAN_CAP = 4096


def _plan_key(checked, args: Mapping, meta: Mapping):
    parts = [id(checked)]
    for k in sorted(meta):
        parts.append((k, meta[k]))
    for k in sorted(args):
        v = args[k]
        if hasattr(v, "shape") and hasattr(v, "stride") and len(v.shape) == 0:
            parts.append((k, float(v.item())))
        elif hasattr(v, "shape") and hasattr(v, "stride"):
            parts.append((k, tuple(v.shape), tuple(v.stride()), getattr(v, "dtype", None),
                          getattr(v, "device", None), type(v)))
        else:
            try:
                parts.append((k, float(v)))
            except (TypeError, ValueError):
                parts.append((k, id(v)))
    return tuple(parts)


def program_writes(checked, args: Mapping, meta: Mapping) -> dict:
    """Per out-parameter, per program, the sorted flat offsets it writes -
    enumerated by the native map VM on the host (ntb_map_enumerate) from the
    same lowered maps the kernels use; the reference collects the same sets
    while simulating (sim.py:288-290, 348)."""
    spec = checked.spec
    binding = _binding(spec, args, meta)
    _, prog = _resolve(checked, allow_generic=True)
    grid = evaluate_grid(checked, binding)
    total = int(np.prod(grid))
    slots = prog.slots(binding)
    out = {}
    for p in spec.params:
        if p.role != "out":
            continue
        rc, offs, mask = _lib.map_enumerate(prog.blob, prog.params.index(p.name), slots)
        if rc:
            raise BackendError(_lib.last_error())
        per = len(offs) // total
        m = mask.astype(bool)
        out[p.name] = [np.sort(offs[i * per:(i + 1) * per][m[i * per:(i + 1) * per]])
                       for i in range(total)]
    return out


def check_write_partition(checked, args: Mapping, meta: Mapping) -> None:
    """sim.check_write_partition twin (sim.py:366-393): per out-parameter the
    programs' writes are pairwise disjoint and cover every element of the
    argument exactly once."""
    writes = program_writes(checked, args, meta)
    for name, per_program in writes.items():
        allo = np.concatenate(per_program) if per_program else np.empty(0, dtype=np.int64)
        if len(np.unique(allo)) != allo.size:
            raise BackendError(f"programs overlap when writing {name!r}(size {allo.size})")
        t = args[name]
        idx = np.zeros(tuple(t.shape), dtype=np.int64)
        for d, (n, st) in enumerate(zip(t.shape, t.stride())):
            shape = [1] * len(t.shape)
            shape[d] = n
            idx = idx + (np.arange(n, dtype=np.int64) * st).reshape(shape)
        if not np.array_equal(np.sort(allo), np.sort(idx.ravel())):
            raise BackendError(f"writes to {name!r} do not cover it exactly: wrote {allo.size} "
                               f"of {idx.size} elements")


def launch(checked, args: Mapping, meta: Mapping, *, stream=None, pid_order: str = "forward",
           collect_writes: bool = False) -> LaunchResult:
    """Execute a CheckedSpec on the current CUDA device (sim.launch twin).

    The first call for a given (spec, shapes, strides, dtype, meta, scalars)
    validates, evaluates checks and grid through the native map VM and
    prebuilds the C-ABI argument block; later calls with the same signature
    only swap the data pointers (host overhead of a few microseconds).
    """
    import torch

    # programs write disjoint outputs (check_write_partition), so their order
    # on the GPU cannot change the result; the reference's knob is accepted
    if pid_order not in ("forward", "reverse"):
        raise LaunchError(f"unknown pid order {pid_order!r}")
    key = _plan_key(checked, args, meta)
    plan = _plans.get(key)
    if plan is None or plan[0] is not checked:
        plan = (checked,) + _make_plan(checked, args, meta)
        if len(_plans) > _PLAN_CAP:
            _plans.clear()
        _plans[key] = plan
    if plan[1] == "jit":
        res = _launch_generated(plan, args, stream)
        return LaunchResult(res.grid, res.total, program_writes(checked, args, meta)) \
            if collect_writes else res
    _, names, kid, dt, n, sizes, strides, ranks, metas, sc, n_sc, result, dev = plan
    ptrs = (ctypes.c_void_p * n)(*[args[nm].data_ptr() for nm in names])
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        rc = _lib.lib().ntb_launch(kid, dt, ptrs, n, sc, n_sc, _lib.i64(sizes), _lib.i64(strides),
                                   ranks, _lib.i64(metas), len(metas), ctypes.c_void_p(stream))
    if rc == _lib.NTB_ERR_UNSUPPORTED:
        raise UnsupportedSpecError(_lib.last_error())
    if rc == _lib.NTB_ERR_ARG or rc == _lib.NTB_ERR_CHECK:
        raise LaunchError(_lib.last_error())
    if rc:
        raise BackendError(_lib.last_error())
    if collect_writes:
        return LaunchResult(result.grid, result.total, program_writes(checked, args, meta))
    return result


def _launch_generated(plan, args: Mapping, stream):
    import torch

    _, _, handle, names, scalars, slots, block, grid_total, result, dev = plan
    store = [ctypes.c_void_p(args[nm].data_ptr()) for nm in names]
    store += [ctypes.c_float(v) for v in scalars]
    ptrs = [ctypes.addressof(c) for c in store] + [slots.ctypes.data]
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        rc = _lib.jit_launch(handle, (grid_total, 1, 1), (block, 1, 1), ptrs, stream)
    if rc:
        raise BackendError(_lib.last_error())
    return result


def _make_generated_plan(checked, binding, prog, grid, args):
    """Generic path: CUDA C++ printed from the spec by
    codegen.py, NVRTC-compiled for sm_100a through the C ABI."""
    import torch

    from . import codegen

    spec = checked.spec
    tensors = [p for p in spec.params if p.rank >= 1]
    ts = [args[p.name] for p in tensors]
    dt = _dtype_code(ts[0]) if isinstance(ts[0], torch.Tensor) else 0
    try:
        gen = codegen.generate(checked, binding, dt)
    except codegen.CodegenError as e:
        raise UnsupportedSpecError(
            f"spec {spec.name!r} matches no sm_100a kernel family and the generic path does not "
            f"cover it: {e}") from None
    for p, t in zip(tensors, ts):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise LaunchError(
                f"argument {p.name!r} must be a CUDA tensor (the B200 backend has no CPU path)")
    for p, t in zip(tensors, ts):
        if _dtype_code(t) != dt or t.device != ts[0].device:
            raise LaunchError(f"argument {p.name!r} must match {ts[0].dtype} on {ts[0].device}")
    with torch.cuda.device(ts[0].device):
        rc, handle = _lib.jit_compile(gen.source, gen.name)
    if rc == _lib.NTB_ERR_UNSUPPORTED:
        raise UnsupportedSpecError(_lib.last_error())
    if rc:
        raise BackendError(_lib.last_error())
    scalars = []
    for p in spec.params:
        if p.rank == 0:
            v = args[p.name]
            scalars.append(float(v.item() if hasattr(v, "item") else v))
    slots = np.array([binding[n] for n in gen.slot_names] or [0], dtype=np.int64)
    total = int(np.prod(grid))
    return ("jit", handle, gen.tensor_params, scalars, slots, gen.block, total,
            LaunchResult(grid=tuple(grid), total=total), ts[0].device)


def _make_plan(checked, args: Mapping, meta: Mapping):
    import torch

    spec = checked.spec
    binding = _binding(spec, args, meta)
    family, prog = _resolve(checked, allow_generic=True)
    rc, grid = _lib.grid_eval(prog.blob, prog.slots(binding))
    if rc == _lib.NTB_ERR_CHECK:
        raise LaunchError(_check_failure(prog, binding))
    if rc == _lib.NTB_ERR_EVAL:
        raise LaunchError(_lib.last_error())
    if rc:
        raise BackendError(_lib.last_error())
    total = int(np.prod(grid))
    if family is None:
        return _make_generated_plan(checked, binding, prog, grid, args)

    tensors = [p for p in spec.params if p.rank >= 1]
    ts = [args[p.name] for p in tensors]
    for p, t in zip(tensors, ts):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise LaunchError(
                f"argument {p.name!r} must be a CUDA tensor (the B200 backend has no CPU path)")
    dt = _dtype_code(ts[0])
    for p, t in zip(tensors, ts):
        if _dtype_code(t) != dt:
            raise LaunchError(f"argument {p.name!r} has dtype {t.dtype}, expected {ts[0].dtype}")
        if t.device != ts[0].device:
            raise LaunchError(f"argument {p.name!r} is on {t.device}, expected {ts[0].device}")
    scalars = []
    for p in spec.params:
        if p.rank == 0:
            v = args[p.name]
            scalars.append(float(v.item() if hasattr(v, "item") else v))
    n = len(ts)
    sizes = np.array([s for t in ts for s in t.shape], dtype=np.int64)
    strides = np.array([s for t in ts for s in t.stride()], dtype=np.int64)
    ranks = (ctypes.c_int * n)(*[t.dim() for t in ts])
    metas = np.array([binding[m] for m in spec.meta], dtype=np.int64)
    sc = (ctypes.c_double * max(1, len(scalars)))(*scalars)
    return ([p.name for p in tensors], _lib.KERNEL_IDS[family], dt, n, sizes, strides, ranks,
            metas, sc, len(scalars), LaunchResult(grid=tuple(grid), total=total), ts[0].device)


def simulate(kernel: str, args: Mapping, meta: Mapping, pid_order: str = "forward",
             dtype=None) -> np.ndarray:
    """GPU twin of the reference's ``verify.simulate`` (verify.py:200-204):
    ``args`` maps every parameter of the catalog kernel to a host numpy
    array (outputs included, as ``verify.make_inputs`` builds them) or a float
    (rank-0 parameters); the arrays go to the current CUDA device as
    ``dtype`` (default float32, the catalog's f32 kind), the kernel runs on
    its native sm_100a path, and the output comes back as numpy."""
    import torch

    dtype = torch.float32 if dtype is None else dtype
    ck = canonical(kernel)
    dev = torch.device("cuda", torch.cuda.current_device())
    targs = {}
    for p in ck.spec.params:
        if p.name not in args:
            raise LaunchError(f"missing argument {p.name!r}")
        v = args[p.name]
        targs[p.name] = float(v) if p.rank == 0 else \
            torch.from_numpy(np.ascontiguousarray(v)).to(dev, dtype)
    launch(ck, targs, meta, pid_order=pid_order)
    outs = [p.name for p in ck.spec.params if p.role == "out"]
    return targs[outs[0]].float().cpu().numpy()


def launch_count() -> int:
    """Kernels launched by libntb200 in this process."""
    return int(_lib.lib().ntb_launch_count())


def path_counts() -> dict:
    """Launches per native execution path (tcgen05 vs generic, ...)."""
    return _lib.path_counts()


# ---- emitted-launcher twins (emit.py:267-293) ------------------------------

def make_launcher(checked):
    spec = checked.spec
    names = [p.name for p in spec.params] + list(spec.meta)
    outs = [p.name for p in spec.params if p.role == "out"]

    def launcher(*a, **kw):
        if len(a) + len(kw) != len(names):
            raise TypeError(f"{spec.name}_launch takes {len(names)} arguments ({', '.join(names)})")
        bound = dict(zip(names, a))
        for k, v in kw.items():
            if k in bound:
                raise TypeError(f"duplicate argument {k!r}")
            bound[k] = v
        args = {p.name: bound[p.name] for p in spec.params}
        meta = {m: bound[m] for m in spec.meta}
        launch(checked, args, meta)
        res = tuple(bound[o] for o in outs)
        return res[0] if len(res) == 1 else res

    launcher.__name__ = f"{spec.name}_launch"
    launcher.__doc__ = f"{spec.name}_launch({', '.join(names)}) on the B200 backend"
    return launcher


def __getattr__(attr):
    # add_launch, mm_launch, ... built on first use
    if attr.endswith("_launch") and attr[: -len("_launch")] in ALL_NAMES:
        fn = make_launcher(canonical(attr[: -len("_launch")]))
        globals()[attr] = fn
        return fn
    raise AttributeError(attr)
