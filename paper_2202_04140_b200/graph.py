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


_HEADER_RE = re.compile(
    r"^ACEDAG v(\d+) group=(T|SO2|O3|O3F) p=(1|2|inf) D=([0-9.]+) numax=(\d+) alg=(orig|gen) n=(\d+)$")


def deserialize_graph(data: bytes) -> EvalGraph:
    """Parse the text format (graphbuild.py:387-464) into a native graph.

    Line-level errors carry byte offsets like the reference; structural
    validation (topological parents, tuple unions, auxiliary flags) is then
    re-checked natively from the parent relation.
    """
    try:
        text = data.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise GraphFormatError("graph data is not valid UTF-8", exc.start) from None
    lines = text.split("\n")
    m = _HEADER_RE.match(lines[0])
    if m is None:
        vm = re.match(r"^ACEDAG v(\d+)\b", lines[0])
        if vm and vm.group(1) != "1":
            raise UnsupportedVersionError(f"unsupported graph format version {vm.group(1)}", 0)
        raise GraphFormatError(f"bad header line: {lines[0]!r}", 0)
    if m.group(1) != "1":
        raise UnsupportedVersionError(f"unsupported graph format version {m.group(1)}", 0)
    group = Group(m.group(2))
    p = math.inf if m.group(3) == "inf" else int(m.group(3))
    try:
        d_raw = float(m.group(4))
    except ValueError:
        raise GraphFormatError(f"bad degree cap {m.group(4)!r}", 0) from None
    spec = DegreeSpec(p, int(d_raw) if d_raw.is_integer() else d_raw)
    numax = int(m.group(5))
    labels = one_particle_indices(group, spec.int_cap())
    lab_index = {e: i for i, e in enumerate(labels)}
    offset = len(lines[0].encode("utf-8")) + 1
    parents, auxes, tuples = [], [], []
    for raw in lines[1:]:
        at = offset
        offset += len(raw.encode("utf-8")) + 1
        if not raw:
            continue
        parts = raw.split(" ")
        if len(parts) not in (4, 5):
            raise GraphFormatError(f"bad node line: {raw!r}", at)
        try:
            ident, aux = int(parts[0]), int(parts[1])
        except ValueError:
            raise GraphFormatError(f"bad node line: {raw!r}", at) from None
        if ident != len(parents):
            raise GraphFormatError(f"node ids must be dense and ascending, got {ident}", at)
        if aux not in (0, 1):
            raise GraphFormatError(f"auxiliary flag must be 0 or 1, got {parts[1]!r}", at)
        try:
            elements = parse_elements(group, parts[2])
        except ValueError as exc:
            raise GraphFormatError(str(exc), at) from None
        if parts[3] == "-":
            if len(parts) != 4:
                raise GraphFormatError(f"bad parent field: {raw!r}", at)
            if len(elements) != 1:
                raise GraphFormatError("only order-1 nodes may lack parents", at)
            par = (-1, -1)
        else:
            if len(parts) != 5:
                raise GraphFormatError(f"bad parent field: {raw!r}", at)
            try:
                par = (int(parts[3]), int(parts[4]))
            except ValueError:
                raise GraphFormatError(f"bad parent ids: {raw!r}", at) from None
            if not all(0 <= q < ident for q in par):
                raise GraphFormatError(f"parent ids must precede node {ident}", at)
            merged = tuple(sorted(tuples[par[0]] + tuples[par[1]]))
            if merged != elements:
                raise GraphFormatError(f"parents do not union to node {ident}", at)
        if len(elements) == 1 and aux:
            raise GraphFormatError("order-1 nodes cannot be auxiliary", at)
        if len(elements) == 1 and (ident >= len(labels) or lab_index.get(elements[0]) != ident):
            raise GraphFormatError(f"order-1 node {ident} out of label order", at)
        tuples.append(elements)
        parents.append(par)
        auxes.append(aux)
    if not parents:
        raise GraphFormatError("graph has no nodes; order-1 seeds are mandatory", offset)
    try:
        return graph_from_parents(group, spec, np.array(parents, np.int32), np.array(auxes, np.uint8),
                                  numax if numax else None, m.group(6), int(m.group(7)))
    except ValueError as exc:
        raise GraphFormatError(str(exc), 0) from None


def write_graph(graph: EvalGraph, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize_graph(graph))


def read_graph(path) -> EvalGraph:
    with open(path, "rb") as fh:
        return deserialize_graph(fh.read())


def format_node(graph: EvalGraph, node: int) -> str:
    return format_elements(graph.elements_of(node))
