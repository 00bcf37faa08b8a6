"""Evaluation path: the reference's evaluator API on sm_100a kernels.

Drop-in functions keep the names, arguments and exceptions of the reference
``acedag.evaluator`` (/root/reference/pkg/src/acedag/evaluator.py):

    one_particle   evaluator.py:61-77     -> K1 (acedag_pool), one particle
    pool           evaluator.py:80-90     -> K1 (acedag_pool)
    evaluate_graph evaluator.py:93-110    -> acedag_eval_nodes (bit-exact)
    naive_eval     evaluator.py:113-121   -> acedag_naive_products (bit-exact)
    evaluate_model evaluator.py:124-142   -> K1 + K2 (acedag_eval)

They move one site across PCIe per call (correct but latency-bound).  The
batched API -- :class:`SitePlan` -- is the production path: device tensors in,
device tensors out, stream-ordered, no host synchronisation.

There is no CPU fallback: without a CUDA device these functions raise.
"""

from __future__ import annotations

import ctypes as C
import math
import random
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .graph import EvalGraph, as_eval_graph
from .indexsets import (Group, DegreeSpec, element_degree, format_elements, one_particle_indices,
                        parse_elements, validate_element)

_NCOORDS = {Group.T: 1, Group.SO2: 2, Group.O3: 3, Group.O3F: 4}

# position workloads (BASELINE cfg3/cfg5): shell radii and cutoff
R_IN, R_CUT = 0.8, 5.0


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2202_04140_b200 evaluates on a CUDA device; none is available "
                           "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev: torch.device | None = None) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _vp(t: torch.Tensor | None) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------- validation

def _check_coords(group: Group, coords) -> None:  # evaluator.py:46-58
    if len(coords) != _NCOORDS[group]:
        raise ValueError(f"{group.value} particles take {_NCOORDS[group]} coordinates, got {coords!r}")
    if group is not Group.T:
        r = coords[0]
        if not 0.0 <= r <= 1.0:
            raise ValueError(f"radius must lie in [0, 1], got {r!r}")
    if group is Group.O3F:
        mu = coords[3]
        if not -1.0 <= mu <= 1.0:
            raise ValueError(f"feature value must lie in [-1, 1], got {mu!r}")


# ----------------------------------------------------------------- batched
# Every device entry point checks its tensors before a pointer crosses the C
# ABI: a wrong dtype, shape or device must be a ValueError, never an
# out-of-bounds access inside a kernel.

def _need(t: torch.Tensor, name: str, dtype, device: torch.device | None = None, shape=None) -> None:
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    dts = dtype if isinstance(dtype, tuple) else (dtype,)
    if t.dtype not in dts:
        raise ValueError(f"{name} must be {' or '.join(str(d) for d in dts)}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _result(result, shape, dtype, device: torch.device) -> torch.Tensor:
    """A caller-supplied output must be a contiguous tensor of exactly the
    output's shape, dtype and device (the kernels write through its pointer)."""
    if result is None:
        return torch.empty(shape, dtype=dtype, device=device)
    _need(result, "result", dtype, device, shape)
    if not result.is_contiguous():
        raise ValueError("result must be contiguous")
    return result


def _counts(counts, S: int, device: torch.device):
    if counts is None:
        return None
    _need(counts, "counts", (torch.int32, torch.int64), device, (S,))
    return counts.to(torch.int32).contiguous()


def pool_batched(group: Group, cap: int, coords: torch.Tensor, counts: torch.Tensor | None = None,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """K1, reference convention.  coords: cuda float64 [S, J, ncoord(group)];
    counts: cuda int32 [S] (ragged sites) or None.  Returns complex128 [S, L]."""
    _need(coords, "coords", torch.float64)
    if coords.dim() != 3 or coords.shape[2] != group.components:
        raise ValueError(f"coords must be [S, J, {group.components}] for {group.value}, got {tuple(coords.shape)}")
    coords = coords.contiguous()
    S, J = coords.shape[0], coords.shape[1]
    L = len(one_particle_indices(group, cap))
    out = _result(out, (S, L), torch.complex128, coords.device)
    counts = _counts(counts, S, coords.device)
    N.check(N.lib().acedag_pool(group.code, int(cap), _vp(coords), _vp(counts), S, J, _vp(out),
                                _stream(coords.device)))
    return out


def pool_positions(cap: int, xyz: torch.Tensor, counts: torch.Tensor | None = None,
                   r_in: float = R_IN, r_cut: float = R_CUT, out: torch.Tensor | None = None):
    """K1 for Cartesian neighbour shells (BASELINE cfg3/cfg5); complex128 [S, L]."""
    _need(xyz, "xyz", torch.float64)
    if xyz.dim() != 3 or xyz.shape[2] != 3:
        raise ValueError(f"xyz must be [S, J, 3], got {tuple(xyz.shape)}")
    xyz = xyz.contiguous()
    S, J = xyz.shape[0], xyz.shape[1]
    L = len(one_particle_indices(Group.O3, cap))
    out = _result(out, (S, L), torch.complex128, xyz.device)
    counts = _counts(counts, S, xyz.device)
    N.check(N.lib().acedag_pool_positions(int(cap), _vp(xyz), _vp(counts), S, J, float(r_in),
                                          float(r_cut), _vp(out), _stream(xyz.device)))
    return out


class SitePlan:
    """A graph compiled for one device, plus the model coefficients.

    ``set_coefficients`` accepts either the reference's dict ``{tuple: c}``
    (evaluate_model's argument) or node ids with a value array ``[T]`` /
    ``[T, n_out]`` (real or complex).  Evaluation entry points take device
    tensors and return device tensors on the current stream.
    """

    def __init__(self, graph, device: int | None = None):
        self.graph: EvalGraph = as_eval_graph(graph)
        if device is None:
            device = _device().index
        self.device = int(device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().acedag_plan_create(self.graph._h, self.device, C.byref(h)))
        self._h = h
        self._dev = torch.device("cuda", self.device)
        self.n_out = 0
        self.complex_coef = False

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and N._lib is not None:
            N._lib.acedag_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    # -- coefficients
    def set_coefficients(self, coefficients=None, node_ids=None, values=None) -> "SitePlan":
        g = self.graph
        if coefficients is not None:
            ids, vals = [], []
            for t, c in coefficients.items():
                i = g.find(t)
                if i < 0:
                    raise KeyError(f"coefficient on tuple absent from the graph: {t!r}")
                if not g.is_target(t):
                    raise ValueError(f"coefficient on non-target node: {t!r}")
                ids.append(i)
                vals.append(complex(c))
            node_ids = np.array(ids, np.int64)
            values = np.array(vals, np.complex128)
        node_ids = np.ascontiguousarray(np.asarray(node_ids, np.int64).reshape(-1))
        values = np.asarray(values)
        if values.ndim == 1:
            values = values[:, None]
        if values.shape[0] != node_ids.shape[0]:
            raise ValueError("node_ids and values disagree in length")
        n_out = values.shape[1]
        cplx = np.iscomplexobj(values) and bool(np.any(values.imag != 0))
        c_re = np.ascontiguousarray(values.real, np.float64)
        c_im = np.ascontiguousarray(values.imag, np.float64) if cplx else None
        with torch.cuda.device(self.device):
            N.check(N.lib().acedag_plan_set_coefficients(self._h, N.ptr(node_ids, C.c_int64),
                                                         N.ptr(c_re, C.c_double), N.ptr(c_im, C.c_double),
                                                         node_ids.shape[0], n_out))
        self.n_out = n_out
        self.complex_coef = cplx
        return self

    def timing(self, enable: bool = True) -> None:
        """Record per-phase CUDA-event timings of subsequent evaluations."""
        N.check(N.lib().acedag_plan_timing(self._h, 1 if enable else 0))

    def read_timing(self) -> dict:
        """Summed device milliseconds per phase since timing() / the last
        read: ``prep`` (tile-major seed copy), ``main`` (the K2 kernel),
        ``post`` (split-tail reduction); ``calls`` evaluations."""
        ms = (C.c_double * 3)()
        calls = C.c_int64()
        N.check(N.lib().acedag_plan_timing_read(self._h, ms, C.byref(calls)))
        return {"prep": ms[0], "main": ms[1], "post": ms[2], "calls": calls.value}

    def kernel_name(self, method: str = "recursive", prec: str = "f64", out: str = "real",
                    sites: int = 1 << 20) -> str:
        """The kernel evaluate() launches for these arguments on ``sites``
        sites (reporting)."""
        return N.lib().acedag_eval_kernel_name(
            self._h, N.METHOD_NAIVE if method == "naive" else N.METHOD_RECURSIVE,
            N.PREC_F32 if prec == "f32" else N.PREC_F64, N.OUT_COMPLEX if out == "complex" else N.OUT_REAL,
            int(sites)).decode()

    def info(self) -> dict:
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib().acedag_plan_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"recursive_products": a.value, "extra_nodes": b.value, "naive_products": c.value,
                "used_seeds": d.value}

    # -- evaluation
    def evaluate(self, A: torch.Tensor, method: str = "recursive", out: str = "real",
                 result: torch.Tensor | None = None) -> torch.Tensor:
        """phi for every site of ``A`` (complex128 [S, L], or complex64 for
        the fp32 recursive mode).  Returns float64 [S] / [S, n_out]
        (``out="real"``) or complex128 (``out="complex"``)."""
        if self.n_out == 0:
            raise ValueError("no coefficients set")
        _need(A, "A", (torch.complex128, torch.complex64), self._dev)
        if A.dim() != 2 or A.shape[1] != self.graph.num_seeds:
            raise ValueError(f"A must be [S, {self.graph.num_seeds}], got {tuple(A.shape)}")
        A = A.contiguous()
        prec = N.PREC_F64 if A.dtype == torch.complex128 else N.PREC_F32
        S = A.shape[0]
        kind = N.OUT_COMPLEX if out == "complex" else N.OUT_REAL
        dt = torch.complex128 if kind == N.OUT_COMPLEX else torch.float64
        shape = (S,) if self.n_out == 1 else (S, self.n_out)
        result = _result(result, shape, dt, self._dev)
        m = N.METHOD_NAIVE if method == "naive" else N.METHOD_RECURSIVE
        N.check(N.lib().acedag_eval(self._h, m, prec, kind, _vp(A), S, _vp(result), _stream(A.device)))
        return result

    def evaluate_host(self, A: torch.Tensor, method: str = "recursive", out: str = "real",
                      result: torch.Tensor | None = None) -> torch.Tensor:
        """End-to-end call on HOST buffers (acedag_eval_host): A is a CPU
        complex128 (or complex64, fp32 recursive mode) tensor [S, L].  Pinned
        A is read in place by the GPU -- only the seed columns the plan uses
        -- pipelined with the kernels; pageable A is copied in row chunks.
        Returns a CPU tensor (pinned unless ``result`` is given) shaped like
        :meth:`evaluate`'s; synchronous.  ``self.last_h2d_bytes`` records the
        input bytes moved to the device."""
        if A.is_cuda:
            raise ValueError("evaluate_host takes a CPU tensor")
        if self.n_out == 0:
            raise ValueError("no coefficients set")
        if A.dim() != 2 or A.shape[1] != self.graph.num_seeds:
            raise ValueError(f"A must be [S, {self.graph.num_seeds}], got {tuple(A.shape)}")
        A = A.contiguous()
        if A.dtype not in (torch.complex128, torch.complex64):
            raise ValueError("A must be complex128 or complex64")
        prec = N.PREC_F64 if A.dtype == torch.complex128 else N.PREC_F32
        S = A.shape[0]
        kind = N.OUT_COMPLEX if out == "complex" else N.OUT_REAL
        dt = torch.complex128 if kind == N.OUT_COMPLEX else torch.float64
        shape = (S,) if self.n_out == 1 else (S, self.n_out)
        if result is None:
            result = torch.empty(shape, dtype=dt, pin_memory=True)
        elif result.is_cuda or result.dtype != dt or tuple(result.shape) != shape or not result.is_contiguous():
            raise ValueError(f"result must be a contiguous CPU {dt} tensor of shape {shape}")
        m = N.METHOD_NAIVE if method == "naive" else N.METHOD_RECURSIVE
        h2d = C.c_int64()
        dev = torch.device("cuda", self.device)
        N.check(N.lib().acedag_eval_host(self._h, m, prec, kind, _vp(A), S, _vp(result), C.byref(h2d),
                                         _stream(dev)))
        self.last_h2d_bytes = h2d.value
        return result

    def evaluate_positions_host(self, xyz: torch.Tensor, r_in: float = R_IN, r_cut: float = R_CUT,
                                chunk: int = 65536, result: torch.Tensor | None = None,
                                sync: bool = True) -> torch.Tensor:
        """End-to-end fused K1 + K2 on a (pinned) host [S, J, 3] tensor."""
        if xyz.is_cuda:
            raise ValueError("evaluate_positions_host takes a CPU tensor")
        return self._host_pipeline(
            xyz, lambda x, r: self.evaluate_positions(x, r_in=r_in, r_cut=r_cut, result=r), chunk, result, sync)

    def _host_pipeline(self, X: torch.Tensor, fn, chunk: int, result, sync: bool):
        """Chunks of X are copied to the device, evaluated by ``fn`` and copied
        back on two streams, so PCIe transfers overlap the kernels.  With
        ``sync`` the host result is complete on return; otherwise it is
        complete once the caller's current stream has drained."""
        S = X.shape[0]
        dev = torch.device("cuda", self.device)
        oshape = () if self.n_out == 1 else (self.n_out,)
        if result is None:
            result = torch.empty((S,) + oshape, dtype=torch.float64, pin_memory=True)
        key = (chunk, X.dtype, tuple(X.shape[1:]), oshape)
        if getattr(self, "_host_ws", (None,))[0] != key:
            self._host_ws = (key, [torch.cuda.Stream(dev) for _ in range(2)],
                             [torch.empty((chunk,) + tuple(X.shape[1:]), dtype=X.dtype, device=dev)
                              for _ in range(2)],
                             [torch.empty((chunk,) + oshape, dtype=torch.float64, device=dev) for _ in range(2)])
        _, streams, bufs, outs = self._host_ws
        caller = torch.cuda.current_stream(dev)
        for s in streams:
            s.wait_stream(caller)
        for i, s0 in enumerate(range(0, S, chunk)):
            n = min(chunk, S - s0)
            st = streams[i % 2]
            with torch.cuda.stream(st):
                bufs[i % 2][:n].copy_(X[s0:s0 + n], non_blocking=True)
                fn(bufs[i % 2][:n], outs[i % 2][:n])
                result[s0:s0 + n].copy_(outs[i % 2][:n], non_blocking=True)
        for s in streams:
            caller.wait_stream(s)
        if sync:
            caller.synchronize()
        return result

    def evaluate_positions(self, xyz: torch.Tensor, counts: torch.Tensor | None = None,
                           r_in: float = R_IN, r_cut: float = R_CUT, out: str = "real",
                           result: torch.Tensor | None = None) -> torch.Tensor:
        """Fused K1 + K2 from Cartesian neighbour vectors [S, J, 3] float64."""
        if self.n_out == 0:
            raise ValueError("no coefficients set")
        _need(xyz, "xyz", torch.float64, self._dev)
        if xyz.dim() != 3 or xyz.shape[2] != 3:
            raise ValueError(f"xyz must be [S, J, 3], got {tuple(xyz.shape)}")
        xyz = xyz.contiguous()
        S, J = xyz.shape[0], xyz.shape[1]
        kind = N.OUT_COMPLEX if out == "complex" else N.OUT_REAL
        dt = torch.complex128 if kind == N.OUT_COMPLEX else torch.float64
        shape = (S,) if self.n_out == 1 else (S, self.n_out)
        result = _result(result, shape, dt, self._dev)
        counts = _counts(counts, S, self._dev)
        N.check(N.lib().acedag_eval_from_positions(self._h, _vp(xyz), _vp(counts), S, J, float(r_in),
                                                   float(r_cut), kind, _vp(result), _stream(xyz.device)))
        return result

    def evaluate_nodes(self, A: torch.Tensor) -> torch.Tensor:
        """All node values, complex128 [S, N], bit-identical to evaluate_graph."""
        _need(A, "A", torch.complex128, self._dev)
        if A.dim() != 2 or A.shape[1] != self.graph.num_seeds:
            raise ValueError("A must be complex128 [S, L]")
        A = A.contiguous()
        S = A.shape[0]
        out = torch.empty((S, self.graph.num_nodes), dtype=torch.complex128, device=A.device)
        N.check(N.lib().acedag_eval_nodes(self._h, _vp(A), S, _vp(out), _stream(A.device)))
        return out

    def reduce_sites(self, phi: torch.Tensor, total: torch.Tensor | None = None) -> torch.Tensor:
        """Deterministic sum over sites of a real phi [S] / [S, n_out]."""
        _need(phi, "phi", torch.float64, self._dev)
        if phi.dim() not in (1, 2) or phi.reshape(phi.shape[0], -1).shape[1] != self.n_out:
            raise ValueError(f"phi must be [S] or [S, {self.n_out}] float64")
        phi = phi.contiguous()
        # the kernel adds into total (callers accumulate several batches)
        total = torch.zeros(self.n_out, dtype=torch.float64, device=self._dev) if total is None else \
            _result(total, (self.n_out,), torch.float64, self._dev)
        N.check(N.lib().acedag_reduce_sites(self._h, _vp(phi), phi.shape[0], _vp(total), _stream(phi.device)))
        return total


def launch_count() -> int:
    """Kernels the native library has launched since it was loaded."""
    return int(N.lib().acedag_launch_count())


def naive_products(vals: torch.Tensor, lens: torch.Tensor | None = None) -> torch.Tensor:
    """Batched naive_eval over rows of complex128 [n, width] (bit-exact);
    lens [n] (each <= width) gives ragged row lengths."""
    _need(vals, "vals", torch.complex128)
    if vals.dim() != 2:
        raise ValueError(f"vals must be [n, width], got {tuple(vals.shape)}")
    vals = vals.contiguous()
    n, w = vals.shape
    out = torch.empty(n, dtype=torch.complex128, device=vals.device)
    if lens is not None:
        _need(lens, "lens", (torch.int32, torch.int64), vals.device, (n,))
        if n and (int(lens.min()) < 0 or int(lens.max()) > w):
            raise ValueError(f"lens must lie in [0, {w}]")
        lens = lens.to(torch.int32).contiguous()
    N.check(N.lib().acedag_naive_products(_vp(vals), _vp(lens), n, w, _vp(out), _stream(vals.device)))
    return out


# ------------------------------------------------------------ drop-ins

def _coords_tensor(group: Group, particles) -> tuple[torch.Tensor, int]:
    for c in particles:
        _check_coords(group, c)
    J = len(particles)
    arr = np.zeros((1, max(J, 1), _NCOORDS[group]), np.float64)
    for j, c in enumerate(particles):
        arr[0, j] = [float(x) for x in c]
    return torch.from_numpy(arr).to(_device()), J


def _pool_array(group: Group, cap: int, particles) -> np.ndarray:
    coords, J = _coords_tensor(group, particles)
    counts = torch.tensor([J], dtype=torch.int32, device=coords.device)
    A = pool_batched(group, cap, coords, counts)
    return A[0].cpu().numpy()


def one_particle(group: Group, element: tuple, coords) -> complex:
    """Value of one basis function for one particle (evaluator.py:61-77)."""
    _check_coords(group, coords)
    validate_element(group, tuple(element))
    cap = element_degree(element)
    labels = one_particle_indices(group, cap)
    A = _pool_array(group, cap, [coords])
    return complex(A[labels.index(tuple(element))])


def pool(group: Group, spec, particles) -> dict[tuple, complex]:
    """Pooled features for every label within the cap (evaluator.py:80-90)."""
    cap = spec.int_cap()
    labels = one_particle_indices(group, cap)
    if not labels:
        return {}
    A = _pool_array(group, cap, particles)
    return {e: complex(v) for e, v in zip(labels, A)}


def _pooled_matrix(g: EvalGraph, pooled) -> np.ndarray:
    A = np.empty((1, g.num_seeds), np.complex128)
    for i, e in enumerate(g.labels):
        try:
            A[0, i] = pooled[e]
        except KeyError:
            raise KeyError(f"pooled basis has no value for one-particle label {e!r}") from None
    return A


def evaluate_graph(graph, pooled: dict) -> list[complex]:
    """Value of every node, by node id (evaluator.py:93-110); bit-exact."""
    g = as_eval_graph(graph)
    A = torch.from_numpy(_pooled_matrix(g, pooled)).to(_device())
    vals = g.plan().evaluate_nodes(A)
    return [complex(v) for v in vals[0].cpu().numpy()]


def naive_eval(elements, pooled: dict) -> complex:
    """Direct product of pooled values over the tuple (evaluator.py:113-121)."""
    row = []
    for e in elements:
        try:
            row.append(pooled[e])
        except KeyError:
            raise KeyError(f"pooled basis has no value for one-particle label {e!r}") from None
    if not row:
        return 1 + 0j
    vals = torch.tensor([row], dtype=torch.complex128, device=_device())
    return complex(naive_products(vals)[0].item())


def evaluate_model(graph, coefficients: dict, particles, real_part: bool = False):
    """sum_k c_k A_k for one configuration (evaluator.py:124-142)."""
    g = as_eval_graph(graph)
    for t in coefficients:  # validation first, like the reference
        if g.find(t) < 0:
            raise KeyError(f"coefficient on tuple absent from the graph: {t!r}")
        if not g.is_target(t):
            raise ValueError(f"coefficient on non-target node: {t!r}")
    dev = _device()
    cap = g.spec.int_cap()
    coords, J = _coords_tensor(g.group, particles)
    counts = torch.tensor([J], dtype=torch.int32, device=dev)
    A = pool_batched(g.group, cap, coords, counts)
    if not coefficients:
        return 0.0 if real_part else 0j
    plan = SitePlan(g, dev.index).set_coefficients(coefficients)
    phi = complex(plan.evaluate(A, out="complex")[0].item())
    plan.close()
    return phi.real if real_part else phi


# ------------------------------------------------- symmetry transforms
# Callers of the path (evaluator.py:149-186): a particle is a coordinate
# tuple whose azimuth sits at a fixed position per group (T: the angle
# itself; SO2: after the radius; O3/O3F: after (r, theta)).

_AZIMUTH = {Group.T: 0, Group.SO2: 1, Group.O3: 2, Group.O3F: 2}


def _shift(coords, pos: int, delta: float) -> tuple:
    c = tuple(coords)
    return c[:pos] + (c[pos] + delta,) + c[pos + 1:]


def rotate_particles(group: Group, particles, alpha: float):
    """Every particle's azimuth advanced by alpha (a z-rotation for O3/O3F)."""
    pos = _AZIMUTH[group]
    return [_shift(c, pos, alpha)[: group.components] for c in particles]


def invert_particles(group: Group, particles):
    """r -> -r: polar angle mirrored, azimuth turned by pi (O3/O3F only)."""
    if not group.has_l:
        raise ValueError(f"inversion applies to O3/O3F, not {group.value}")
    out = []
    for c in particles:
        c = tuple(c)
        out.append((c[0], math.pi - c[1], c[2] + math.pi) + c[3:group.components])
    return out


def random_particles(group: Group, rng: random.Random, max_count: int = 8):
    """1..max_count random particles, drawing from ``rng`` in the reference's
    order (count, then per particle: radius, cos(theta), azimuth, feature as
    the group has them) so a seeded rng reproduces its configurations."""
    two_pi = 2.0 * math.pi
    draws = {
        Group.T: lambda: (rng.uniform(0.0, two_pi),),
        Group.SO2: lambda: (rng.random(), rng.uniform(0.0, two_pi)),
        Group.O3: lambda: (rng.random(), math.acos(rng.uniform(-1.0, 1.0)), rng.uniform(0.0, two_pi)),
    }
    draws[Group.O3F] = lambda: draws[Group.O3]() + (rng.uniform(-1.0, 1.0),)
    n = rng.randint(1, max_count)
    return [draws[group]() for _ in range(n)]


@dataclass(frozen=True)
class InvarianceReport:
    group: Group
    trials: int
    rotation_max_dev: float
    inversion_max_dev: float | None


def invariance_check(group: Group, graph, particles, trials: int = 8, seed: int = 0) -> InvarianceReport:
    """Target-node deviations under rotations/inversion (evaluator.py:201-224),
    all transformed configurations evaluated as one batch of sites."""
    g = as_eval_graph(graph)
    rng = random.Random(seed)
    confs = [list(particles)]
    for _ in range(trials):
        confs.append(rotate_particles(group, particles, rng.uniform(0.0, 2.0 * math.pi)))
    if group.has_l:
        confs.append(invert_particles(group, particles))
    dev = _device()
    J = max(1, len(particles))
    arr = np.zeros((len(confs), J, _NCOORDS[group]))
    for s, conf in enumerate(confs):
        for j, c in enumerate(conf):
            arr[s, j] = c
    counts = torch.full((len(confs),), len(particles), dtype=torch.int32, device=dev)
    A = pool_batched(group, g.spec.int_cap(), torch.from_numpy(arr).to(dev), counts)
    vals = g.plan(dev.index).evaluate_nodes(A)[:, torch.as_tensor(g.target_ids, device=dev)]
    base = vals[0]
    dev_all = (vals - base).abs() / (1.0 + base.abs())
    rot = float(dev_all[1:trials + 1].max().item()) if trials and vals.shape[1] else 0.0
    inv = None
    if group.has_l:
        inv = float(dev_all[trials + 1].max().item()) if vals.shape[1] else 0.0
    return InvarianceReport(group, trials, rot, inv)


# ------------------------------------------------------------ file formats
# Particle and coefficient text files (evaluator.py:231-290), callers of the
# path kept for the CLI: UTF-8, one record per line, blank lines skipped.
# Error texts follow the reference's (the CLI prints them).

def _records(path, comments: bool):
    """(line number, raw line, stripped line) of every non-blank line;
    with ``comments`` '#' lines are yielded too (the caller decides)."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    for no, raw in enumerate(text.splitlines(), start=1):
        body = raw.strip()
        if body and (comments or not body.startswith("#")):
            yield no, raw, body


def write_particles(path, group: Group, particles) -> None:
    rows = [f"# group={group.value}"]
    for coords in particles:
        _check_coords(group, coords)
        rows.append(" ".join(repr(float(x)) for x in coords))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(rows) + "\n")


def read_particles(path):
    """``# group=<G>`` header, then one whitespace-separated particle per line."""
    group, particles = None, []
    for no, raw, body in _records(path, comments=True):
        if body[0] == "#":
            key, _, val = body.lstrip("#").strip().partition("=")
            if key == "group" and _ == "=":
                group = Group(val.strip())
            continue
        if group is None:
            raise ValueError(f"{path}: missing '# group=...' header before data")
        try:
            coords = tuple(map(float, body.split()))
        except ValueError:
            raise ValueError(f"{path}:{no}: bad coordinate line: {raw!r}") from None
        _check_coords(group, coords)
        particles.append(coords)
    if group is None:
        raise ValueError(f"{path}: missing '# group=...' header")
    return group, particles


def write_coefficients(path, coefficients: dict) -> None:
    rows = []
    for t in sorted(coefficients):
        z = complex(coefficients[t])
        rows.append(f"{format_elements(t)} {z.real!r} {z.imag!r}\n")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("".join(rows))


def read_coefficients(path, group: Group) -> dict:
    """``<tuple> <re> <im>`` per line; '#' lines are comments."""
    coefs = {}
    for no, raw, body in _records(path, comments=False):
        fields = body.split()
        if len(fields) != 3:
            raise ValueError(f"{path}:{no}: expected '<tuple> <re> <im>', got {raw!r}")
        key = parse_elements(group, fields[0])
        try:
            re_, im_ = float(fields[1]), float(fields[2])
        except ValueError:
            raise ValueError(f"{path}:{no}: bad coefficient values: {raw!r}") from None
        coefs[key] = complex(re_, im_)
    return coefs
