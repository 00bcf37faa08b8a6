"""Graph-file reader cases, answered by the REFERENCE's deserialize_graph.

Runs where /root/reference is mounted; writes graph_format_cases.json, which
tests/test_graph_format.py replays against the native reader
(csrc/graph_io.cpp).  Each case is a byte string derived from a small
reference-built graph by one edit; the reference's outcome is recorded as
("ok", sha256 of its re-serialization) or (exception type, str(exc), offset).

    python tests/golden/make_golden_format.py
"""

from __future__ import annotations

import base64
import hashlib
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from acedag.graphbuild import build_graph, deserialize_graph, serialize_graph  # noqa: E402
from acedag.indexsets import DegreeSpec, Group  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    out = []
    for grp, D, nu, alg, n in (("O3", 4, 3, "orig", 1), ("SO2", 4, 3, "gen", 2), ("T", 3, 4, "orig", 1),
                               ("O3F", 3, 3, "orig", 1)):
        g = build_graph(Group(grp), DegreeSpec(1, D), nu, alg, n)
        out.append((f"valid {grp}", serialize_graph(g)))
    base = serialize_graph(build_graph(Group.O3, DegreeSpec(1, 4), 3))
    lines = base.decode().split("\n")
    hdr, body = lines[0], lines[1:]
    L = sum(k * k for k in range(1, 6))  # len(one_particle_indices(O3, 4)) = 55
    first_prod = L + 1

    def edit(i, new):
        ls = list(lines)
        ls[i] = new
        return "\n".join(ls).encode()

    prod = lines[first_prod]
    pid, paux, pel, pa, pb = prod.split(" ")
    seed = lines[1]
    out += [
        ("not utf8", base[:200] + b"\xff" + base[200:]),
        ("truncated utf8", base[:120] + b"\xe2\x82"),
        ("overlong utf8", base[:90] + b"\xc0\xaf" + base[90:]),
        ("surrogate utf8", base[:90] + b"\xed\xa0\x80" + base[90:]),
        ("bad magic", edit(0, hdr.replace("ACEDAG", "ACEDAX"))),
        ("version 2", edit(0, hdr.replace("v1", "v2"))),
        ("version 01", edit(0, hdr.replace("v1", "v01"))),
        ("version 2 garbage", edit(0, "ACEDAG v2 whatever")),
        ("version 2x", edit(0, "ACEDAG v2x whatever")),
        ("header trailing space", edit(0, hdr + " ")),
        ("header cr", edit(0, hdr + "\r")),
        ("bad group", edit(0, hdr.replace("group=O3", "group=O4"))),
        ("bad p", edit(0, hdr.replace("p=1", "p=3"))),
        ("degree 1.2.3", edit(0, hdr.replace("D=4", "D=1.2.3"))),
        ("degree dot", edit(0, hdr.replace("D=4", "D=."))),
        ("degree 4.", edit(0, hdr.replace("D=4", "D=4."))),
        ("degree 4.5", edit(0, hdr.replace("D=4", "D=4.5"))),
        ("numax 0", edit(0, hdr.replace("numax=3", "numax=0"))),
        ("header only", (hdr + "\n").encode()),
        ("header no newline", hdr.encode()),
        ("empty", b""),
        ("three fields", edit(3, " ".join(lines[3].split(" ")[:3]))),
        ("six fields", edit(first_prod, prod + " 7")),
        ("double space", edit(3, lines[3].replace(" ", "  ", 1))),
        ("id not int", edit(3, "x" + lines[3][1:])),
        ("aux not int", edit(3, lines[3].replace(" 0 ", " z ", 1))),
        ("aux 2", edit(3, lines[3].replace(" 0 ", " 2 ", 1))),
        ("aux +1 on seed", edit(3, lines[3].replace(" 0 ", " +1 ", 1))),
        ("id skipped", edit(3, "3" + lines[3][1:])),
        ("id padded", edit(3, " 2" + lines[3][1:].replace(" ", "\t", 0))),
        ("id underscore", edit(11, "1_0" + lines[11][2:])),
        ("id double underscore", edit(11, "1__0" + lines[11][2:])),
        ("elements not int", edit(1, "0 0 0,a,0 -")),
        ("elements count", edit(1, "0 0 0,0 -")),
        ("elements spaced int", edit(1, "0 0 0,+0, 0 -")),
        ("elements empty", edit(3, "2 0  -")),
        ("elements negative n", edit(3, "2 0 -1,0,0 -")),
        ("elements m above l", edit(3, "2 0 0,1,2 -")),
        ("elements order", edit(first_prod, f"{pid} {paux} 1,0,0,0,0,0 {pa} {pb}")),
        ("seed with parents dash extra", edit(3, lines[3] + " 1")),
        ("product without parents", edit(first_prod, f"{pid} {paux} {pel} -")),
        ("parent ids not int", edit(first_prod, f"{pid} {paux} {pel} {pa} q")),
        ("parent id not preceding", edit(first_prod, f"{pid} {paux} {pel} {pa} {pid}")),
        ("parent id negative", edit(first_prod, f"{pid} {paux} {pel} -1 {pb}")),
        ("parents do not union", edit(first_prod, f"{pid} {paux} {pel} 0 1")),
        ("seed aux", edit(3, lines[3].replace(" 0 ", " 1 ", 1))),
        ("aux inconsistent", edit(first_prod, f"{pid} {1 - int(paux)} {pel} {pa} {pb}")),
        ("duplicate tuple", "\n".join(lines[:first_prod + 1] + [f"{first_prod} {paux} {pel} {pa} {pb}"]
                                      + [""]).encode()),
        ("crlf", base.replace(b"\n", b"\r\n")),
        ("blank lines", base.replace(b"\n", b"\n\n", 5)),
        ("seed outside the cap (restriction)", edit(1, "0 0 5,0,0 -")),
        ("seeds out of order (restriction)", edit(1, lines[2].replace("1 ", "0 ", 1))),
    ]
    return out


def main():
    res = []
    for name, data in cases():
        try:
            g = deserialize_graph(data)
            res.append({"name": name, "data": base64.b64encode(data).decode(), "ok": True,
                        "sha256": hashlib.sha256(serialize_graph(g)).hexdigest(), "nodes": len(g.nodes)})
        except Exception as exc:  # noqa: BLE001 -- the reference's outcome is the fixture
            res.append({"name": name, "data": base64.b64encode(data).decode(), "ok": False,
                        "type": type(exc).__name__, "message": str(exc), "offset": getattr(exc, "offset", None)})
    with open(os.path.join(HERE, "graph_format_cases.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(len(res), "cases")


if __name__ == "__main__":
    main()
