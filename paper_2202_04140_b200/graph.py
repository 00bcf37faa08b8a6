"""Recursive-evaluation DAG on the host, built natively.

``build_graph`` runs the reference's Algorithm 1 / Algorithm 2 insertion
(graphbuild.py:139-268) in C++ (csrc/graph.cpp); the result is byte-identical
under ``serialize_graph`` (graphbuild.py:374-384; SHA-256 pins in
tests/golden).  The graph is held as SoA arrays -- parent pairs, auxiliary
flags, orders -- which is the form the device plan compiler consumes; the
reference's per-node ``GraphNode`` objects are materialised lazily for API
compatibility only.
"""

from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _native as N
from .indexsets import (DegreeSpec, Group, format_elements, one_particle_indices, parse_elements,
                        satisfies_constraints)

ALGORITHMS = ("orig", "gen")


class GraphFormatError(ValueError):
    """Malformed graph file; ``offset`` is the byte position of the bad line."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at byte {offset})")
        self.offset = offset


class UnsupportedVersionError(GraphFormatError):
    pass


@dataclass(frozen=True)
class GraphNode:
    id: int
    elements: tuple
    parents: tuple | None
    auxiliary: bool

    @property
    def order(self) -> int:
        return len(self.elements)


class EvalGraph:
    """DAG of basis tuples with dense, topological ids (graphbuild.py:76-123).

    Owns a native handle; ``parents`` [N, 2] int32 (-1 for seeds), ``aux``
    [N] bool, ``order`` [N] int32 and ``target_ids`` are numpy views of it.
    """

    def __init__(self, handle, group: Group, spec: DegreeSpec, nu_max, alg: str, n: int):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.group = group
        self.spec = spec
        self.nu_max = nu_max
        self.alg = alg
        self.n = n
        lib = N.lib()
        nn, ns, nt, na, mo = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        N.check(lib.acedag_graph_info(self._h, C.byref(nn), C.byref(ns), C.byref(nt), C.byref(na), C.byref(mo)))
        self.num_nodes, self.num_seeds, self.num_targets = nn.value, ns.value, nt.value
        self.num_aux, self.max_order = na.value, mo.value
        par = np.empty((self.num_nodes, 2), np.int32)
        aux = np.empty(self.num_nodes, np.uint8)
        order = np.empty(self.num_nodes, np.int32)
        tgt = np.empty(max(1, self.num_targets), np.int32)
        N.check(lib.acedag_graph_arrays(self._h, N.ptr(par, C.c_int32), N.ptr(aux, C.c_uint8),
                                        N.ptr(order, C.c_int32), N.ptr(tgt, C.c_int32)))
        self.parents = par
        self.aux = aux.astype(bool)
        self.order = order
        self.target_ids = tgt[: self.num_targets].astype(np.int64)
        self.labels = one_particle_indices(group, spec.int_cap())
        self._label_index = {e: i for i, e in enumerate(self.labels)}
        self._nodes = None
        self._plans = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N._lib is not None:
            for p in getattr(self, "_plans", {}).values():
                p.close()
            N._lib.acedag_graph_destroy(h)
            self._h = None

    # -- container behaviour (graphbuild.py:95-117)
    def __len__(self) -> int:
        return self.num_nodes

    def __contains__(self, elements) -> bool:
        return self.find(elements) >= 0

    def __iter__(self) -> Iterator[GraphNode]:
        return iter(self.nodes)

    def seed_ids(self, elements) -> list[int] | None:
        try:
            ids = sorted(self._label_index[e] for e in elements)
        except (KeyError, TypeError):
            return None
        return ids

    def find(self, elements) -> int:
        ids = self.seed_ids(tuple(elements))
        if not ids or len(ids) > 8:
            return -1
        arr = np.array(ids, np.int32)
        return int(N.lib().acedag_graph_find(self._h, N.ptr(arr, C.c_int32), len(ids)))

    def id_of(self, elements) -> int:
        i = self.find(elements)
        if i < 0:
            raise KeyError(tuple(elements))
        return i

    def is_target(self, elements) -> bool:
        if self.nu_max is not None and len(elements) > self.nu_max:
            return False
        return satisfies_constraints(elements, self.group) and self.spec.within(elements)

    def elements_of(self, node: int) -> tuple:
        buf = np.empty(8, np.int32)
        k = N.check(N.lib().acedag_graph_node_seeds(self._h, int(node), N.ptr(buf, C.c_int32), 8))
        return tuple(self.labels[i] for i in buf[:k])

    @property
    def nodes(self) -> list[GraphNode]:
        """Reference-style node list (built on first use)."""
        if self._nodes is None:
            out = []
            for i in range(self.num_nodes):
                a, b = self.parents[i]
                out.append(GraphNode(i, self.elements_of(i), None if a < 0 else (int(a), int(b)),
                                     bool(self.aux[i])))
            self._nodes = out
        return self._nodes

    def plan(self, device: int | None = None):
        """Device plan for this graph (cached per device)."""
        from .evaluator import SitePlan
        import torch
        dev = torch.cuda.current_device() if device is None else int(device)
        p = self._plans.get(dev)
        if p is None:
            p = self._plans[dev] = SitePlan(self, device=dev)
        return p


def _handle_to_graph(h, group, spec, nu_max, alg, n) -> EvalGraph:
    return EvalGraph(h, group, spec, nu_max, alg, n)


def build_graph(group: Group, spec: DegreeSpec, nu_max: int, alg: str = "orig", n: int = 1) -> EvalGraph:
    """All invariant tuples of order <= nu_max (graphbuild.py:243-268), natively."""
    if nu_max < 1:
        raise ValueError(f"nu_max must be >= 1, got {nu_max!r}")
    if alg not in ALGORITHMS:
        raise ValueError(f"alg must be one of {ALGORITHMS}, got {alg!r}")
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n!r}")
    if alg == "orig":
        n = 1
    h = C.c_void_p()
    N.check(N.lib().acedag_graph_build(group.code, spec.p_code, float(spec.max_degree), int(nu_max),
                                       ALGORITHMS.index(alg), int(n), C.byref(h)))
    return EvalGraph(h, group, spec, nu_max, alg, n)


def seed_graph(group: Group, spec: DegreeSpec, nu_max: int | None = None) -> EvalGraph:
    """Only the order-1 nodes (graphbuild.py:236-240)."""
    L = len(one_particle_indices(group, spec.int_cap()))
    par = np.full((L, 2), -1, np.int32)
    return graph_from_parents(group, spec, par, nu_max=nu_max)


def graph_from_parents(group: Group, spec: DegreeSpec, parents, aux=None, nu_max=None, alg="orig",
                       n: int = 1) -> EvalGraph:
    """Wrap an externally built DAG given its parent pairs [N, 2]."""
    par = np.ascontiguousarray(np.asarray(parents, np.int32).reshape(-1, 2))
    L = len(one_particle_indices(group, spec.int_cap()))
    auxa = None if aux is None else np.ascontiguousarray(np.asarray(aux, np.uint8))
    h = C.c_void_p()
    N.check(N.lib().acedag_graph_from_parents(group.code, spec.p_code, float(spec.max_degree),
                                              int(nu_max or 0), ALGORITHMS.index(alg), int(n),
                                              par.shape[0], L, N.ptr(par, C.c_int32),
                                              N.ptr(auxa, C.c_uint8), C.byref(h)))
    return EvalGraph(h, group, spec, nu_max, alg, n)


def as_eval_graph(graph) -> EvalGraph:
    """Accept this package's EvalGraph or a reference ``acedag`` EvalGraph
    (duck-typed: ``group``, ``spec``, ``nu_max``, ``nodes[i].parents``)."""
    if isinstance(graph, EvalGraph):
        return graph
    cached = getattr(graph, "_b200_graph", None)
    if cached is not None and cached.num_nodes == len(graph.nodes):
        return cached
    group = Group(graph.group.value)
    spec = DegreeSpec(graph.spec.p, graph.spec.max_degree)
    par = np.array([n.parents if n.parents is not None else (-1, -1) for n in graph.nodes], np.int32)
    aux = np.array([n.auxiliary for n in graph.nodes], np.uint8)
    g = graph_from_parents(group, spec, par, aux, graph.nu_max, getattr(graph, "alg", "orig"),
                           getattr(graph, "n", 1))
    try:
        graph._b200_graph = g
    except AttributeError:
        pass
    return g


def serialize_graph(graph: EvalGraph) -> bytes:
    """Versioned text format, byte-identical to graphbuild.py:374-384."""
    g = as_eval_graph(graph)
    n = C.c_int64(0)
    lib = N.lib()
    N.check(lib.acedag_graph_serialize(g._h, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    N.check(lib.acedag_graph_serialize(g._h, buf, C.byref(n)))
    return buf.raw[: n.value]


# violation kinds of acedag_graph_deserialize (include/acedag_b200.h ACEDAG_GE_*)
(_GE_NOT_UTF8, _GE_VERSION, _GE_HEADER, _GE_DEGREE, _GE_NODE_LINE, _GE_NOT_DENSE, _GE_AUX_FLAG, _GE_ELEMENTS,
 _GE_PARENT_FIELD, _GE_ORPHAN, _GE_PARENT_IDS, _GE_PARENT_ORDER, _GE_UNION, _GE_SEED_AUX, _GE_AUX_MISMATCH,
 _GE_DUPLICATE, _GE_EMPTY, _GE_SEED_LAYOUT, _GE_LIMIT) = range(1, 20)


def _format_error(kind: int, offset: int, line: str, group: Group | None, native_msg: str) -> GraphFormatError:
    """The reference's exception for a violation the native reader found
    (graphbuild.py:387-464 wording), composed from the offending line."""
    fields = line.split(" ")
    if kind == _GE_NOT_UTF8:
        return GraphFormatError("graph data is not valid UTF-8", offset)
    if kind == _GE_VERSION:
        version = re.match(r"ACEDAG v(\d+)", line)[1]
        return UnsupportedVersionError(f"unsupported graph format version {version}", 0)
    if kind == _GE_HEADER:
        return GraphFormatError(f"bad header line: {line!r}", 0)
    if kind == _GE_DEGREE:
        degree = re.search(r" D=([0-9.]+) ", line)[1]
        return GraphFormatError(f"bad degree cap {degree!r}", 0)
    quoted = {_GE_NODE_LINE: "bad node line", _GE_PARENT_FIELD: "bad parent field", _GE_PARENT_IDS: "bad parent ids"}
    if kind in quoted:
        return GraphFormatError(f"{quoted[kind]}: {line!r}", offset)
    if kind == _GE_AUX_FLAG:
        return GraphFormatError(f"auxiliary flag must be 0 or 1, got {fields[1]!r}", offset)
    if kind == _GE_ELEMENTS:
        try:
            parse_elements(group, fields[2])
        except ValueError as exc:
            return GraphFormatError(str(exc), offset)
        return GraphFormatError(f"tuple components must be ASCII integers in this build: {fields[2]!r}", offset)
    per_node = {_GE_NOT_DENSE: "node ids must be dense and ascending, got", _GE_PARENT_ORDER: "parent ids must precede node",
                _GE_UNION: "parents do not union to node", _GE_AUX_MISMATCH: "auxiliary flag inconsistent on node",
                _GE_DUPLICATE: "duplicate tuple at node"}
    if kind in per_node:
        return GraphFormatError(f"{per_node[kind]} {int(fields[0])}", offset)
    fixed = {_GE_ORPHAN: "only order-1 nodes may lack parents", _GE_SEED_AUX: "order-1 nodes cannot be auxiliary",
             _GE_EMPTY: "graph has no nodes; order-1 seeds are mandatory"}
    if kind in fixed:
        return GraphFormatError(fixed[kind], offset)
    # this build's own limits (seed layout, order <= 8): the native text
    return GraphFormatError(native_msg.rsplit(" (at byte", 1)[0], offset)


def deserialize_graph(data: bytes) -> EvalGraph:
    """Read the versioned text format (graphbuild.py:387-464) natively
    (csrc/graph_io.cpp: one pass, checks in the reference's order, byte
    offsets like the reference's); errors are the reference's exception types
    and messages."""
    data = bytes(data)
    lib = N.lib()
    h = C.c_void_p()
    kind, off, ls, ln = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
    rc = lib.acedag_graph_deserialize(data, len(data), C.byref(h), C.byref(kind), C.byref(off), C.byref(ls),
                                      C.byref(ln))
    if rc == N.EFORMAT:
        line = data[ls.value: ls.value + ln.value].decode("utf-8", "replace")
        group = None
        m = re.match(r"ACEDAG v\d+ group=(T|SO2|O3|O3F) ", data[:256].decode("utf-8", "replace"))
        if m:
            group = Group(m[1])
        raise _format_error(kind.value, off.value, line, group, N.last_error())
    N.check(rc)
    grp, p, nu, alg, n = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    D = C.c_double()
    N.check(lib.acedag_graph_spec(h, C.byref(grp), C.byref(p), C.byref(D), C.byref(nu), C.byref(alg), C.byref(n)))
    d = D.value
    spec = DegreeSpec(math.inf if p.value == 0 else p.value, int(d) if float(d).is_integer() else d)
    group = (Group.T, Group.SO2, Group.O3, Group.O3F)[grp.value]
    return EvalGraph(h, group, spec, nu.value or None, ALGORITHMS[alg.value], n.value)


def write_graph(graph: EvalGraph, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize_graph(graph))


def read_graph(path) -> EvalGraph:
    with open(path, "rb") as fh:
        return deserialize_graph(fh.read())


def format_node(graph: EvalGraph, node: int) -> str:
    return format_elements(graph.elements_of(node))
