"""Basis specification on the host: symmetry groups, one-particle labels,
degree rules and the tuple text syntax.

Mirrors the public surface of the reference's ``acedag.indexsets``
(/root/reference/pkg/src/acedag/indexsets.py) that the evaluation path needs:
the label order produced by :func:`one_particle_indices` IS the column layout
of every pooled-basis matrix ``A[S, L]`` the kernels consume
(indexsets.py:170-191), and :func:`satisfies_constraints` /
:meth:`DegreeSpec.within` decide which tuples may carry a coefficient
(indexsets.py:137-163).  Tuple enumeration itself runs natively inside the
graph builder (csrc/graph.cpp).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction


class Group(Enum):
    """Symmetry group of the basis (indexsets.py:37-52)."""

    T = "T"
    SO2 = "SO2"
    O3 = "O3"
    O3F = "O3F"

    @property
    def components(self) -> int:
        return {"T": 1, "SO2": 2, "O3": 3, "O3F": 4}[self.value]

    @property
    def has_l(self) -> bool:
        return self.value in ("O3", "O3F")

    @property
    def code(self) -> int:
        """Integer code of the C ABI (ACEDAG_GROUP_*)."""
        return ("T", "SO2", "O3", "O3F").index(self.value)


def _m_index(arity: int) -> int:
    return 0 if arity == 1 else (1 if arity == 2 else 2)


def element_m(element: tuple) -> int:
    return element[_m_index(len(element))]


def element_l(element: tuple) -> int:
    return element[1] if len(element) >= 3 else 0


def element_degree(element: tuple) -> int:
    """|m| (T), n+|m| (SO2), n+l (O3), n+l+f (O3F) -- indexsets.py:70-79."""
    k = len(element)
    if k == 1:
        return abs(element[0])
    if k == 2:
        return element[0] + abs(element[1])
    return element[0] + element[1] + (element[3] if k == 4 else 0)


def validate_element(group: Group, element) -> None:
    """ValueError unless ``element`` is a label of ``group`` (indexsets.py:82-97)."""
    if not isinstance(element, tuple) or len(element) != group.components:
        raise ValueError(f"{group.value} labels have {group.components} components, got {element!r}")
    if not all(isinstance(c, int) for c in element):
        raise ValueError(f"label components must be integers, got {element!r}")
    if group is Group.SO2 and element[0] < 0:
        raise ValueError(f"radial degree must be non-negative in {element!r}")
    if group.has_l:
        if element[0] < 0 or element[1] < 0:
            raise ValueError(f"n and l must be non-negative in {element!r}")
        if abs(element[2]) > element[1]:
            raise ValueError(f"|m| <= l violated in {element!r}")
        if group is Group.O3F and element[3] < 0:
            raise ValueError(f"feature degree must be non-negative in {element!r}")


def canonical(elements) -> tuple:
    return tuple(sorted(elements))


def is_canonical(elements) -> bool:
    return all(a <= b for a, b in zip(elements, elements[1:]))


@dataclass(frozen=True)
class DegreeSpec:
    """p-norm degree cap (indexsets.py:109-146); exact integer membership."""

    p: float
    max_degree: float

    def __post_init__(self):
        if self.p not in (1, 2, math.inf):
            raise ValueError(f"p must be 1, 2 or inf, got {self.p!r}")
        if not (self.max_degree >= 0 and math.isfinite(self.max_degree)):
            raise ValueError(f"max_degree must be a finite non-negative number, got {self.max_degree!r}")

    @property
    def p_code(self) -> int:
        """C ABI encoding: 1, 2, or 0 for inf."""
        return 0 if self.p == math.inf else int(self.p)

    def int_cap(self) -> int:
        return math.floor(self.max_degree)

    def power_cap(self) -> int:
        return math.floor(Fraction(self.max_degree) ** 2) if self.p == 2 else math.floor(self.max_degree)

    def power_key(self, elements) -> int:
        degs = [element_degree(e) for e in elements]
        if self.p == 1:
            return sum(degs)
        if self.p == 2:
            return sum(d * d for d in degs)
        return max(degs, default=0)

    def within(self, elements) -> bool:
        return self.power_key(elements) <= self.power_cap()


def tuple_degree(elements, spec: DegreeSpec):
    key = spec.power_key(elements)
    return math.sqrt(key) if spec.p == 2 else key


def satisfies_constraints(elements, group: Group) -> bool:
    """Zero m-sum, and even l-sum for O3/O3F (indexsets.py:157-163)."""
    if sum(element_m(e) for e in elements):
        return False
    return not (group.has_l and sum(element_l(e) for e in elements) % 2)


def one_particle_indices(group: Group, max_degree: int) -> list[tuple]:
    """Labels with element degree <= cap, in canonical (= A column) order."""
    cap = int(max_degree)
    if cap < 0:
        return []
    if group is Group.T:
        return [(m,) for m in range(-cap, cap + 1)]
    out: list[tuple] = []
    for n in range(cap + 1):
        if group is Group.SO2:
            out += [(n, m) for m in range(n - cap, cap - n + 1)]
            continue
        for l in range(cap - n + 1):
            for m in range(-l, l + 1):
                if group is Group.O3:
                    out.append((n, l, m))
                else:
                    out += [(n, l, m, f) for f in range(cap - n - l + 1)]
    return out


def format_elements(elements) -> str:
    """``-1,0,1``-style component list (indexsets.py:434-436)."""
    return ",".join(str(c) for e in elements for c in e)


def parse_elements(group: Group, text: str) -> tuple:
    """Inverse of :func:`format_elements` with validation (indexsets.py:439-453)."""
    try:
        comps = [int(tok) for tok in text.split(",")]
    except ValueError:
        raise ValueError(f"tuple components must be integers: {text!r}") from None
    k = group.components
    if not comps or len(comps) % k:
        raise ValueError(f"expected a multiple of {k} components for {group.value}, got {len(comps)}")
    elements = tuple(tuple(comps[i:i + k]) for i in range(0, len(comps), k))
    for e in elements:
        validate_element(group, e)
    if not is_canonical(elements):
        raise ValueError(f"tuple is not in canonical (sorted) order: {text!r}")
    return elements
