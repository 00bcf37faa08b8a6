"""CPU ORACLE for the acedag evaluation path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain Python + NumPy, the reference algorithm of
``acedag`` (arXiv 2202.04140 reference, mounted read-only at
/root/reference/pkg/src/acedag) for the hot path named by BASELINE.json's
north_star: pooling of the one-particle basis, recursive evaluation of the
product DAG, the naive product oracle and the linear model sum, together with
the host-side DAG construction whose output the kernels consume.

It exists only as the CHECKER.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg (``cpu_baseline`` / ``--impl reference``)
may import it.  The product package ``paper_2202_04140_b200`` never imports
anything from ``oracle/`` and fails loudly when its CUDA library is missing.

Parity pins (see tests/test_oracle_golden.py and tests/golden/):
  * graph construction: SHA-256 of the serialized graph equals the reference's
    ``serialize_graph(build_graph(...))`` for every golden build, including
    the survey-pinned BASELINE configs (cfg1, cfg2/3 -- SURVEY.md 8c);
  * node values: bit-identical to ``evaluate_graph`` on the committed golden
    inputs (no-FMA complex products, CPython ``_Py_c_prod`` formula);
  * pool / one_particle: golden vectors produced by the reference itself
    (tests/golden/make_golden.py, run in the container that has the reference).

Function-by-function citations refer to /root/reference/pkg/src/acedag/*.py.
"""

from __future__ import annotations

import cmath
import hashlib
import itertools
import math
from fractions import Fraction

import numpy as np

# ---------------------------------------------------------------------------
# Index algebra  (indexsets.py)

GROUPS = ("T", "SO2", "O3", "O3F")
NCOMP = {"T": 1, "SO2": 2, "O3": 3, "O3F": 4}          # indexsets.py:55
_MPOS = {1: 0, 2: 1, 3: 2, 4: 2}                       # indexsets.py:58


def group_has_l(group: str) -> bool:                   # indexsets.py:50-52
    return group in ("O3", "O3F")


def element_m(e) -> int:                               # indexsets.py:61-62
    return e[_MPOS[len(e)]]


def element_l(e) -> int:                               # indexsets.py:65-67
    return e[1] if len(e) >= 3 else 0


def element_degree(e) -> int:                          # indexsets.py:70-79
    k = len(e)
    if k == 1:
        return abs(e[0])
    if k == 2:
        return e[0] + abs(e[1])
    if k == 3:
        return e[0] + e[1]
    return e[0] + e[1] + e[3]


class Spec:
    """Degree rule (indexsets.py:109-146): p in {1, 2, inf}, cap D."""

    def __init__(self, p, max_degree):
        if p not in (1, 2, math.inf):
            raise ValueError(f"p must be 1, 2 or inf, got {p!r}")
        self.p = p
        self.max_degree = max_degree

    def int_cap(self) -> int:                          # indexsets.py:127-129
        return math.floor(self.max_degree)

    def power_cap(self) -> int:                        # indexsets.py:131-135
        if self.p == 2:
            return math.floor(Fraction(self.max_degree) ** 2)
        return math.floor(self.max_degree)

    def power_key(self, elements) -> int:              # indexsets.py:137-143
        degs = [element_degree(e) for e in elements]
        if self.p == 1:
            return sum(degs)
        if self.p == 2:
            return sum(d * d for d in degs)
        return max(degs, default=0)

    def within(self, elements) -> bool:                # indexsets.py:145-146
        return self.power_key(elements) <= self.power_cap()


def satisfies_constraints(elements, group: str) -> bool:   # indexsets.py:157-163
    if sum(element_m(e) for e in elements) != 0:
        return False
    return not (group_has_l(group) and sum(element_l(e) for e in elements) % 2)


def one_particle_indices(group: str, cap: int) -> list[tuple]:   # indexsets.py:170-191
    cap = int(cap)
    if cap < 0:
        return []
    if group == "T":
        return [(m,) for m in range(-cap, cap + 1)]
    if group == "SO2":
        return [(n, m) for n in range(cap + 1) for m in range(-(cap - n), cap - n + 1)]
    if group == "O3":
        return [(n, l, m) for n in range(cap + 1) for l in range(cap - n + 1)
                for m in range(-l, l + 1)]
    return [(n, l, m, f) for n in range(cap + 1) for l in range(cap - n + 1)
            for m in range(-l, l + 1) for f in range(cap - n - l + 1)]


def enumerate_tuples(group: str, order: int, spec: Spec) -> list[tuple]:
    """Set of canonical invariant tuples (indexsets.py:368-388).

    The reference uses pruned per-group generators; only the resulting SET
    matters to the graph build because ``build_graph`` re-sorts the targets
    (graphbuild.py:259-260).  This walker prunes on the exact remaining
    power budget and on the m-sum reachability bound |M| <= remaining degree,
    valid for p=1 because every label's degree is >= |m|.
    """
    labels = one_particle_indices(group, spec.int_cap())
    degs = [element_degree(e) for e in labels]
    ms = [element_m(e) for e in labels]
    ls = [element_l(e) for e in labels]
    cap = spec.int_cap()
    pcap = spec.power_cap()
    out: list[tuple] = []
    pre: list[int] = []

    def cost(d):
        return d if spec.p == 1 else (d * d if spec.p == 2 else 0)

    def rec(i0, rem, msum, lsum, slots):
        if slots == 0:
            if msum == 0 and (not group_has_l(group) or lsum % 2 == 0):
                out.append(tuple(labels[i] for i in pre))
            return
        for i in range(i0, len(labels)):
            c = cost(degs[i])
            if c > rem:
                continue
            nm = msum + ms[i]
            left = rem - c
            if spec.p == 1:
                if abs(nm) > left:
                    continue
            elif abs(nm) > (slots - 1) * cap:
                continue
            pre.append(i)
            rec(i, left, nm, lsum + ls[i], slots - 1)
            pre.pop()

    if order == 1:
        return [(e,) for e in labels if element_m(e) == 0
                and (not group_has_l(group) or element_l(e) % 2 == 0)]
    rec(0, pcap if spec.p != math.inf else 0, 0, 0, order)
    return out


# ---------------------------------------------------------------------------
# Splits  (dependency.py:38-60)

def proper_splits(elements) -> list[tuple[tuple, tuple]]:
    groups = [(e, len(list(g))) for e, g in itertools.groupby(elements)]
    res = []
    for counts in itertools.product(*[range(c + 1) for _, c in groups]):
        left, right = [], []
        for (e, c), j in zip(groups, counts):
            left += [e] * j
            right += [e] * (c - j)
        if left and right:
            pair = (tuple(left), tuple(right))
            if pair[0] <= pair[1]:
                res.append(pair)
    res.sort()
    return res


# ---------------------------------------------------------------------------
# Graph construction  (graphbuild.py:76-268)

class OracleGraph:
    """Flat restatement of EvalGraph: parallel lists keyed by dense id."""

    def __init__(self, group: str, spec: Spec, nu_max, alg="orig", n=1):
        if alg not in ("orig", "gen"):
            raise ValueError(f"alg must be one of ('orig', 'gen'), got {alg!r}")
        self.group, self.spec, self.nu_max, self.alg, self.n = group, spec, nu_max, alg, n
        self.elements: list[tuple] = []
        self.parents: list = []
        self.aux: list[bool] = []
        self.ids: dict[tuple, int] = {}

    def is_target(self, t) -> bool:                    # graphbuild.py:119-123
        if self.nu_max is not None and len(t) > self.nu_max:
            return False
        return satisfies_constraints(t, self.group) and self.spec.within(t)

    def add(self, t, parents) -> int:                  # graphbuild.py:132-137
        nid = len(self.elements)
        self.elements.append(t)
        self.parents.append(parents)
        self.aux.append(False if len(t) == 1 else not self.is_target(t))
        self.ids[t] = nid
        return nid

    def seed(self):                                    # graphbuild.py:127-130
        for e in one_particle_indices(self.group, self.spec.int_cap()):
            self.add((e,), None)

    def present_split(self, t):                        # graphbuild.py:139-148
        for left, right in proper_splits(t):
            a = self.ids.get(left)
            if a is not None:
                b = self.ids.get(right)
                if b is not None:
                    return a, b
        return None

    def insert_original(self, t) -> int:               # graphbuild.py:150-167
        t = tuple(t)
        if t in self.ids:
            return self.ids[t]
        if len(t) == 1:
            raise ValueError(f"one-particle label outside the seeded range: {t!r}")
        par = self.present_split(t)
        if par is not None:
            return self.add(t, par)
        head = max(t, key=lambda e: (element_degree(e), e))
        rest = list(t)
        rest.remove(head)
        self.insert_original(tuple(rest))
        return self.insert_original(t)

    def insert_generalized(self, t, n) -> int:         # graphbuild.py:169-187
        t = tuple(t)
        if t in self.ids:
            return self.ids[t]
        if len(t) == 1:
            raise ValueError(f"one-particle label outside the seeded range: {t!r}")
        par = self.present_split(t)
        if par is not None:
            return self.add(t, par)
        size = min(n, len(t) - 1)
        best, best_key = None, -1                      # graphbuild.py:189-202
        for block in set(itertools.combinations(t, size)):
            k = self.spec.power_key(block)
            if k > best_key or (k == best_key and block > best):
                best, best_key = block, k
        rest = list(t)
        for e in best:
            rest.remove(e)
        self.insert_original(best)
        self.insert_generalized(tuple(rest), n)
        return self.insert_generalized(t, n)


def build_graph(group: str, spec: Spec, nu_max: int, alg="orig", n=1) -> OracleGraph:
    """graphbuild.py:243-268 -- targets by order, then (power_key, tuple)."""
    if nu_max < 1:
        raise ValueError(f"nu_max must be >= 1, got {nu_max!r}")
    if alg == "orig":
        n = 1
    g = OracleGraph(group, spec, nu_max, alg, n)
    g.seed()
    for order in range(2, nu_max + 1):
        targets = enumerate_tuples(group, order, spec)
        targets.sort(key=lambda t: (spec.power_key(t), t))
        for t in targets:
            if alg == "orig":
                g.insert_original(t)
            else:
                g.insert_generalized(t, n)
    return g


def _fmt_number(x) -> str:                             # graphbuild.py:369-371
    xf = float(x)
    return str(int(xf)) if xf.is_integer() else repr(xf)


def serialize_graph(g: OracleGraph) -> bytes:          # graphbuild.py:374-384
    p = "inf" if g.spec.p == math.inf else str(int(g.spec.p))
    lines = [f"ACEDAG v1 group={g.group} p={p} D={_fmt_number(g.spec.max_degree)} "
             f"numax={g.nu_max or 0} alg={g.alg} n={g.n}"]
    for i, (t, par, aux) in enumerate(zip(g.elements, g.parents, g.aux)):
        comps = ",".join(str(c) for e in t for c in e)
        ps = f"{par[0]} {par[1]}" if par else "-"
        lines.append(f"{i} {int(aux)} {comps} {ps}")
    return ("\n".join(lines) + "\n").encode("utf-8")


def graph_sha256(g: OracleGraph) -> str:
    return hashlib.sha256(serialize_graph(g)).hexdigest()


def graph_arrays(g: OracleGraph):
    """SoA view: parent arrays (-1 for seeds), aux flags, target ids (id order)."""
    n = len(g.elements)
    pa = np.full(n, -1, np.int64)
    pb = np.full(n, -1, np.int64)
    for i, par in enumerate(g.parents):
        if par is not None:
            pa[i], pb[i] = par
    aux = np.array(g.aux, bool)
    targets = np.array([i for i, t in enumerate(g.elements)
                        if not g.aux[i] and g.is_target(t)], np.int64)
    return pa, pb, aux, targets


# ---------------------------------------------------------------------------
# Special functions  (special.py:19-63)

def chebyshev(k: int, x: float) -> float:              # special.py:19-28
    if k < 0:
        raise ValueError("degree must be non-negative")
    if k == 0:
        return 1.0
    prev, cur = 1.0, x
    for _ in range(k - 1):
        prev, cur = cur, 2.0 * x * cur - prev
    return cur


def legendre_assoc(l: int, m: int, x: float) -> float:    # special.py:31-47
    if not 0 <= m <= l:
        raise ValueError(f"need 0 <= m <= l, got l={l}, m={m}")
    s = math.sqrt(max(0.0, (1.0 - x) * (1.0 + x)))
    p0 = 1.0
    for k in range(1, m + 1):
        p0 *= -(2 * k - 1) * s
    if l == m:
        return p0
    p1 = x * (2 * m + 1) * p0
    for ll in range(m + 2, l + 1):
        p0, p1 = p1, (x * (2 * ll - 1) * p1 - (ll + m - 1) * p0) / (ll - m)
    return p1


def sph_harm(l: int, m: int, theta: float, phi: float) -> complex:   # special.py:50-63
    if abs(m) > l:
        raise ValueError(f"need |m| <= l, got l={l}, m={m}")
    am = abs(m)
    norm = math.sqrt((2 * l + 1) / (4.0 * math.pi)
                     * float(Fraction(math.factorial(l - am), math.factorial(l + am))))
    y = norm * legendre_assoc(l, am, math.cos(theta)) * cmath.exp(1j * am * phi)
    if m < 0:
        y = (-1) ** am * y.conjugate()
    return y


# ---------------------------------------------------------------------------
# One-particle basis, pooling  (evaluator.py:43-90)

def check_coords(group: str, c) -> None:               # evaluator.py:46-58
    if len(c) != NCOMP[group]:
        raise ValueError(f"{group} particles take {NCOMP[group]} coordinates, got {c!r}")
    if group != "T" and not 0.0 <= c[0] <= 1.0:
        raise ValueError(f"radius must lie in [0, 1], got {c[0]!r}")
    if group == "O3F" and not -1.0 <= c[3] <= 1.0:
        raise ValueError(f"feature value must lie in [-1, 1], got {c[3]!r}")


def one_particle(group: str, e, c) -> complex:         # evaluator.py:61-77
    check_coords(group, c)
    if group == "T":
        return cmath.exp(1j * e[0] * c[0])
    if group == "SO2":
        return chebyshev(e[0], 2.0 * c[0] - 1.0) * cmath.exp(-1j * e[1] * c[1])
    val = chebyshev(e[0], 2.0 * c[0] - 1.0) * sph_harm(e[1], e[2], c[1], c[2])
    if group == "O3F":
        val = val * chebyshev(e[3], c[3])
    return val


def pool(group: str, spec: Spec, particles) -> list[complex]:
    """evaluator.py:80-90, as a list in one_particle_indices order."""
    out = []
    for e in one_particle_indices(group, spec.int_cap()):
        acc = 0j
        for c in particles:
            acc = acc + one_particle(group, e, c)
        out.append(acc)
    return out


# Position workloads (BASELINE cfg3/cfg5).  The reference takes spherical
# coordinates with r in [0, 1] and has no cutoff (evaluator.py:51-54,70,74);
# these are the builder's stated extensions,
# applied AROUND the reference's one_particle -- parity of the cutoff itself
# is by construction, not pinned by the reference.
R_IN, R_CUT = 0.8, 5.0


def cutoff_weight(r: float) -> float:
    """f_c(r) = (1 + cos(pi r / r_c)) / 2 for r < r_c, else 0."""
    return 0.5 * (1.0 + math.cos(math.pi * r / R_CUT)) if r < R_CUT else 0.0


def cartesian_to_particle(x: float, y: float, z: float):
    r = math.sqrt(x * x + y * y + z * z)
    xs = min(1.0, max(0.0, (r - R_IN) / (R_CUT - R_IN)))
    theta = math.acos(max(-1.0, min(1.0, z / r)))
    phi = math.atan2(y, x)
    return r, (xs, theta, phi)


def pool_positions(cap: int, xyz: np.ndarray) -> list[complex]:
    """A_k = sum_j f_c(r_j) * one_particle(O3, k, (x_j, theta_j, phi_j))."""
    parts = [cartesian_to_particle(*map(float, p)) for p in xyz]
    out = []
    for e in one_particle_indices("O3", cap):
        acc = 0j
        for r, c in parts:
            acc = acc + cutoff_weight(r) * one_particle("O3", e, c)
        out.append(acc)
    return out


# ---------------------------------------------------------------------------
# Recursive and naive evaluation, model sum  (evaluator.py:93-142)

def evaluate_nodes(pa: np.ndarray, pb: np.ndarray, A: np.ndarray):
    """evaluator.py:93-110 over a batch of sites, node-major.

    ``A`` is complex [S, L] in one_particle_indices order.  Returns (re, im),
    each float64 [N, S].  Each product uses CPython's ``_Py_c_prod`` formula
    (re = ar*br - ai*bi, im = ar*bi + ai*br) with separate roundings (NumPy
    does not contract to FMA), so every node is bit-identical to
    ``evaluate_graph``.
    """
    n = len(pa)
    S, L = A.shape
    re = np.empty((n, S))
    im = np.empty((n, S))
    re[:L] = A.real.T
    im[:L] = A.imag.T
    for k in range(L, n):
        a, b = pa[k], pb[k]
        ar, ai, br, bi = re[a], im[a], re[b], im[b]
        re[k] = ar * br - ai * bi
        im[k] = ar * bi + ai * br
    return re, im


def model_sum(re, im, target_ids, coeffs_re, coeffs_im=None):
    """evaluator.py:141: sequential sum from 0j of c * v in coefficient order."""
    S = re.shape[1]
    acc_r = np.zeros(S)
    acc_i = np.zeros(S)
    cim = np.zeros(len(target_ids)) if coeffs_im is None else coeffs_im
    for t, cr, ci in zip(target_ids, coeffs_re, cim):
        vr, vi = re[t], im[t]
        acc_r = acc_r + (cr * vr - ci * vi)
        acc_i = acc_i + (cr * vi + ci * vr)
    return acc_r, acc_i


def naive_products(tuples_as_ids, A: np.ndarray):
    """evaluator.py:113-121: left-to-right product from 1+0j, per tuple."""
    S = A.shape[0]
    re = np.empty((len(tuples_as_ids), S))
    im = np.empty((len(tuples_as_ids), S))
    for r, ids in enumerate(tuples_as_ids):
        orr = np.ones(S)
        oi = np.zeros(S)
        for i in ids:
            br, bi = A[:, i].real, A[:, i].imag
            orr, oi = orr * br - oi * bi, orr * bi + oi * br
        re[r], im[r] = orr, oi
    return re, im


def energy_scale(re, target_ids, coeffs_re):
    """Sigma_k |c_k Re A_k| per site -- the normalisation of the fp64 parity gate."""
    s = np.zeros(re.shape[1])
    for t, c in zip(target_ids, coeffs_re):
        s += np.abs(c * re[t])
    return s
