"""`#pragma hdarray` frontend (optional half).

The paper's frontend "parse[s] OpenCL kernel functions and HDArray pragmas, collect[s]
... use and def offset information, that is written to the file M ... used to
initialize the HDArray table, and generate[s] code for HDArray pragmas and directives
that pass partitioning information to the runtime".  Here:

* ``parse(source)`` reads kernel sources (OpenCL ``__kernel`` or CUDA ``__global__``)
  and host sources, and returns the file-M table: for every annotated kernel its
  parameter list and the clauses of Table 1 — ``use(X,(o,...))`` /
  ``def(X,(o,...))`` offsets (``*`` = the whole extent), ``use@(X)`` /
  ``def@(X)`` absolute-section markers — and every
  ``partition(ID, (extents), dev:d, (start,length)..., ...)`` clause (Listing 1,
  P:L199-201; (start, length) per reading R2).
* ``write_file_m`` / ``load_file_m``: the table as JSON.
* ``Program``: the host side of ``HDArrayApplyKernel("name", part, args...)``
  (P:L229-231): binds a file-M kernel to one of the library's built-in kernels and maps
  the source's parameter order to the C-ABI's, so a call passes the arguments in the
  kernel's own order.  Absolute sections come from ``set_absolute_use/def`` and
  ``set_trapezoid_use/def`` (Table 2) before the call.

Host logic only: offsets are handed to ``hda_apply`` unchanged; composing them with the
work partition, planning and moving data all happen in the library.
"""
from __future__ import annotations

import json
import re

from .hdarray import STAR, trapezoid

_PRAGMA = re.compile(r"^\s*#\s*pragma\s+hdarray\b(.*)$", re.IGNORECASE)
_KERNEL = re.compile(r"(?:__kernel|__global__)\s+(?:[\w:<>\s\*]*?\s)?(\w+)\s*\(([^)]*)\)", re.S)
_CLAUSE = re.compile(r"(use@|def@|use|def|partition)\s*\(", re.IGNORECASE)


class PragmaError(ValueError):
    pass


def _join_continuations(src: str):
    out, cur = [], ""
    for line in src.splitlines():
        s = line.rstrip()
        if s.endswith("\\"):
            cur += s[:-1] + " "
            continue
        out.append(cur + s)
        cur = ""
    if cur:
        out.append(cur)
    return out


def _balanced(text: str, i: int):
    """text[i] == '(' -> (inner text, index after the matching ')')."""
    depth = 0
    for j in range(i, len(text)):
        if text[j] == "(":
            depth += 1
        elif text[j] == ")":
            depth -= 1
            if depth == 0:
                return text[i + 1:j], j + 1
    raise PragmaError(f"unbalanced parentheses in: {text.strip()}")


def _offset(tok: str):
    tok = tok.strip()
    if tok == "*":
        return "*"
    if not re.fullmatch(r"[+-]?\d+", tok):
        raise PragmaError(f"bad offset component {tok!r} (an integer or '*', P:L186)")
    return int(tok)


def _tuple(text: str):
    text = text.strip()
    if not (text.startswith("(") and text.endswith(")")):
        raise PragmaError(f"expected an offset tuple, got {text!r}")
    return tuple(_offset(t) for t in text[1:-1].split(","))


def _split_top(text: str):
    """split on commas at parenthesis depth 0."""
    parts, depth, cur = [], 0, ""
    for ch in text:
        if ch == "," and depth == 0:
            parts.append(cur)
            cur = ""
            continue
        depth += ch == "("
        depth -= ch == ")"
        cur += ch
    if cur.strip():
        parts.append(cur)
    return [p.strip() for p in parts]


def _clauses(body: str):
    i, out = 0, []
    while i < len(body):
        m = _CLAUSE.search(body, i)
        if not m:
            if body[i:].strip():
                raise PragmaError(f"unrecognised text in pragma: {body[i:].strip()!r}")
            break
        if body[i:m.start()].strip():
            raise PragmaError(f"unrecognised text in pragma: {body[i:m.start()].strip()!r}")
        inner, i = _balanced(body, m.end() - 1)
        out.append((m.group(1).lower(), inner))
    return out


def _params(text: str):
    ps = []
    for p in _split_top(text):
        if not p:
            continue
        name = re.findall(r"\w+", p)[-1]
        ps.append({"name": name, "array": "*" in p or "[" in p})
    return ps


def _partition(inner: str):
    items = _split_top(inner)
    if len(items) < 2:
        raise PragmaError("partition(ID, (extents), dev:d, (start,len)...)")
    pid = items[0]
    domain = tuple(int(v) for v in _tuple(items[1]))
    nd = len(domain)
    devs, cur = {}, None
    for it in items[2:]:
        m = re.fullmatch(r"dev\s*:\s*(\d+)\s*(.*)", it, re.S)
        if m:
            cur = int(m.group(1))
            if cur in devs:
                raise PragmaError(f"partition {pid}: dev:{cur} given twice")
            devs[cur] = []
            it = m.group(2).strip()
            if not it:
                continue
        if cur is None:
            raise PragmaError(f"partition {pid}: region before any dev:")
        st, ln = _tuple(it)
        devs[cur].append((int(st), int(ln)))
    P = len(devs)
    if sorted(devs) != list(range(P)):
        raise PragmaError(f"partition {pid}: devices must be 0..{P - 1}")
    lb, ub = [], []
    for d in range(P):
        if len(devs[d]) != nd:
            raise PragmaError(f"partition {pid}: dev:{d} needs {nd} (start,length) pairs")
        lb.append([s for s, _ in devs[d]])
        ub.append([s + n for s, n in devs[d]])  # (start, length), reading R2
    return pid, {"domain": list(domain), "lb": lb, "ub": ub}


def parse(source: str) -> dict:
    """file-M table of one or more sources (kernels and host code)."""
    lines = _join_continuations(source)
    fm = {"kernels": {}, "partitions": {}}
    pending = None  # clauses of a kernel pragma waiting for its kernel
    for k, line in enumerate(lines):
        m = _PRAGMA.match(line)
        if m:
            cl = _clauses(m.group(1))
            kern = [(c, t) for c, t in cl if c != "partition"]
            for c, t in cl:
                if c == "partition":
                    pid, part = _partition(t)
                    if pid in fm["partitions"]:
                        raise PragmaError(f"partition {pid} declared twice")
                    fm["partitions"][pid] = part
            if kern:
                if pending is not None:
                    raise PragmaError("two kernel pragmas without a kernel between them")
                pending = kern
            continue
        if pending is not None and line.strip():
            rest = "\n".join(lines[k:])
            km = _KERNEL.search(rest)
            if not km or not re.fullmatch(r'((extern\s*"C"|static|inline)\s*)*', rest[:km.start()].strip()):
                raise PragmaError(f"a kernel pragma must precede a kernel definition (line {k + 1})")
            name, params = km.group(1), _params(km.group(2))
            arrays = {p["name"] for p in params if p["array"]}
            acc = {}
            for c, t in pending:
                items = _split_top(t)
                arr = items[0]
                if arr not in arrays:
                    raise PragmaError(f"kernel {name}: {c}({arr},...) names no array parameter")
                a = acc.setdefault(arr, {"use": [], "def": [], "use_abs": False, "def_abs": False})
                if c in ("use@", "def@"):
                    if len(items) != 1:
                        raise PragmaError(f"kernel {name}: {c}({arr}) takes only the array (P:L189)")
                    a[c[:3] + "_abs"] = True
                    continue
                if len(items) < 2:
                    raise PragmaError(f"kernel {name}: {c}({arr}) needs an offset tuple")
                for tup in items[1:]:
                    o = _tuple(tup)
                    if o not in a[c]:
                        a[c].append(o)
            if name in fm["kernels"]:
                raise PragmaError(f"kernel {name} annotated twice")
            fm["kernels"][name] = {"params": params, "access": acc}
            pending = None
    if pending is not None:
        raise PragmaError("kernel pragma at the end of the source without a kernel")
    return fm


def write_file_m(fm: dict, path: str) -> None:
    with open(path, "w") as f:
        json.dump(fm, f, indent=1, sort_keys=True)


def load_file_m(path: str) -> dict:
    with open(path) as f:
        fm = json.load(f)
    for k in fm["kernels"].values():
        for a in k["access"].values():
            a["use"] = [tuple(o) for o in a["use"]]
            a["def"] = [tuple(o) for o in a["def"]]
    return fm


def _abi(o):
    return tuple(STAR if v == "*" else int(v) for v in o)


class Program:
    """Host side of HDArrayApplyKernel over a file-M table and an HDArray context."""

    def __init__(self, h, fm: dict):
        self.h, self.fm = h, fm
        self.binds = {}
        self.parts = {}
        self.abs = {}  # (kernel, part) -> {param: {"use": [[boxes] per dev], "def": ...}}

    def bind(self, kernel: str, kernel_id: int, arrays, scalars=()):
        """kernel_id: a built-in (H.K_*); arrays / scalars: the source's parameter names
        in the C-ABI's positional order (include/hdarray.h lists it per kernel)."""
        if kernel not in self.fm["kernels"]:
            raise KeyError(f"kernel {kernel} not in file M")
        names = {p["name"] for p in self.fm["kernels"][kernel]["params"]}
        for n in list(arrays) + list(scalars):
            if n not in names:
                raise KeyError(f"kernel {kernel} has no parameter {n}")
        self.binds[kernel] = (kernel_id, list(arrays), list(scalars))

    def partition(self, pid: str):
        """the manual partition a `partition` clause declared (expanded to a call that
        returns a partition ID)."""
        if pid not in self.parts:
            p = self.fm["partitions"][pid]
            self.parts[pid] = self.h.partition_manual(p["domain"], p["lb"], p["ub"])
        return self.parts[pid]

    def _abs_slot(self, kernel, part, param, what):
        acc = self.fm["kernels"][kernel]["access"].get(param)
        if acc is None or not acc[what + "_abs"]:
            raise KeyError(f"kernel {kernel}: {param} has no {what}@ clause")
        slot = self.abs.setdefault((kernel, part), {}).setdefault(
            param, {"use": [[] for _ in range(self.h.P)], "def": [[] for _ in range(self.h.P)]})
        return slot[what]

    def set_absolute_use(self, kernel, part, param, dev, lb, ub):
        """HDArraySetAbsoluteUse (Table 2): one more absolute box of `param` used by
        device `dev` (half-open [lb, ub), reading R1)."""
        self._abs_slot(kernel, part, param, "use")[dev].append((tuple(lb), tuple(ub)))

    def set_absolute_def(self, kernel, part, param, dev, lb, ub):
        self._abs_slot(kernel, part, param, "def")[dev].append((tuple(lb), tuple(ub)))

    def set_trapezoid_use(self, kernel, part, param, dev, corners):
        """HDArraySetTrapezoidUse (Table 2): corners [(top,ul),(top,ur),(bottom,bl),
        (bottom,br)]; the row bands the library's hda_trapezoid rasterises (reading R20)
        become absolute use boxes."""
        self._abs_slot(kernel, part, param, "use")[dev].extend(trapezoid(corners))

    def set_trapezoid_def(self, kernel, part, param, dev, corners):
        self._abs_slot(kernel, part, param, "def")[dev].extend(trapezoid(corners))

    def apply_kernel(self, kernel: str, part, *args):
        """HDArrayApplyKernel(kName, partID, args...) with args in the kernel source's
        parameter order (arrays as HDArray handles, scalars as numbers)."""
        if kernel not in self.binds:
            raise KeyError(f"kernel {kernel} is not bound to a built-in (Program.bind)")
        k = self.fm["kernels"][kernel]
        params = k["params"]
        if len(args) != len(params):
            raise TypeError(f"{kernel} takes {len(params)} arguments, got {len(args)}")
        val = {p["name"]: a for p, a in zip(params, args)}
        kid, arrays, scalars = self.binds[kernel]
        accs = [k["access"].get(n, {"use": [], "def": [], "use_abs": False, "def_abs": False}) for n in arrays]
        absolute = [a["use_abs"] or a["def_abs"] for a in accs]
        sc = [val[n] for n in scalars]
        if not any(absolute):
            acc = [(val[n], [_abi(o) for o in a["use"]], [_abi(o) for o in a["def"]]) for n, a in zip(arrays, accs)]
            return self.h.apply(kid, part, acc, sc)
        if not all(absolute) or any(a["use"] or a["def"] for a in accs):
            raise ValueError(f"kernel {kernel}: mixing offset and absolute clauses in one call is not supported")
        slots = self.abs.get((kernel, part), {})
        empty = [[] for _ in range(self.h.P)]
        acc = [(val[n], slots.get(n, {}).get("use", empty), slots.get(n, {}).get("def", empty)) for n in arrays]
        return self.h.apply_abs(kid, part, acc, sc)


def _cname(s: str) -> str:
    return re.sub(r"\W", "_", s)


def emit_c(fm: dict) -> str:
    """Task (3) of the paper's frontend: the file-M table as C for host
    programs written against include/hdarray.h — per offset-annotated kernel an
    access-list builder in the kernel's array-parameter order, per `partition`
    clause a function that creates the manual partition (hda_partition_manual)."""
    out = ["/* generated by paper_1809_05657_b200.frontend from #pragma hdarray clauses */",
           "#include <stdint.h>", '#include "hdarray.h"', ""]
    for name, k in fm["kernels"].items():
        arrays = [p["name"] for p in k["params"] if p["array"]]
        accs = [k["access"].get(a, {"use": [], "def": [], "use_abs": False, "def_abs": False}) for a in arrays]
        if any(a["use_abs"] or a["def_abs"] for a in accs):
            out.append(f"/* kernel {name}: absolute sections (use@/def@) — build hda_abs_access_t at run time */")
            out.append("")
            continue
        cn = _cname(name)
        for a, acc in zip(arrays, accs):
            for kind in ("use", "def"):
                flat = [("HDA_STAR" if v == "*" else str(int(v))) for t in acc[kind] for v in t]
                body = ", ".join(flat) if flat else "0"
                out.append(f"static const int32_t hdam_{cn}_{_cname(a)}_{kind}[] = {{{body}}};")
        out.append(f"/* kernel {name}: arrays in parameter order: {', '.join(arrays)} */")
        out.append(f"static inline int32_t hdam_{cn}_n_arrays(void) {{ return {len(arrays)}; }}")
        out.append(f"static inline void hdam_{cn}_access(hda_access_t* acc, const hda_array_t* arrays) {{")
        for i, (a, acc) in enumerate(zip(arrays, accs)):
            ca = _cname(a)
            out.append(f"  acc[{i}].array = arrays[{i}];")
            out.append(f"  acc[{i}].n_use = {len(acc['use'])};")
            out.append(f"  acc[{i}].use = hdam_{cn}_{ca}_use;")
            out.append(f"  acc[{i}].n_def = {len(acc['def'])};")
            out.append(f"  acc[{i}].def = hdam_{cn}_{ca}_def;")
        out.append("}")
        out.append("")
    for pid, p in fm["partitions"].items():
        nd, P = len(p["domain"]), len(p["lb"])
        dom = ", ".join(str(v) for v in p["domain"])
        lbs = ", ".join(str(v) for row in p["lb"] for v in row)
        ubs = ", ".join(str(v) for row in p["ub"] for v in row)
        out.append(f"/* partition {pid}: {P} devices, (start, length) pairs read as R2 */")
        out.append(f"static inline int hdam_partition_{_cname(pid)}(hda_ctx_t* ctx, hda_part_t* out) {{")
        out.append(f"  static const int64_t dom[] = {{{dom}}}, lbs[] = {{{lbs}}}, ubs[] = {{{ubs}}};")
        out.append(f"  return hda_partition_manual(ctx, {nd}, dom, lbs, ubs, out);")
        out.append("}")
        out.append("")
    return "\n".join(out)
