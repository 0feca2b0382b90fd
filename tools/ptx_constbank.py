#!/usr/bin/env python3
"""PTX pass: move 64-bit floating-point immediates into one constant-bank table.

ptxas materialises every f64 immediate whose low 32 bits are not zero with two
UMOVs (one per 32-bit half) before the instruction that reads it; in the ORd
reaction kernel those moves are ~13% of the executed warp instructions
(profiles/r02c_react_c4_digest.txt). Reading the same constants from a
`.const` table lets ptxas use LDCU.64 / LDCU.128 (one instruction per one or
two constants, uniform registers). Values and arithmetic are unchanged, so
the results are bit-identical.

usage: ptx_constbank.py in.ptx out.ptx
"""
import re
import sys

IMM = re.compile(r"\b0d([0-9A-Fa-f]{16})\b")
FUNC_OPEN = re.compile(r"^\s*(\.visible\s+|\.weak\s+)?(\.entry|\.func)\b")


def transform(src: str) -> tuple[str, int, int]:
    lines = src.split("\n")
    table: dict[str, int] = {}
    out: list[str] = []
    in_func = False
    depth = 0
    nreg = 0  # registers used in the current function
    decl_at = -1
    uses = 0

    def slot(h: str) -> int:
        h = h.upper()
        if h not in table:
            table[h] = len(table)
        return table[h]

    for ln in lines:
        if not in_func and FUNC_OPEN.match(ln):
            in_func, depth, nreg, decl_at = True, 0, 0, -1
        if in_func:
            opens, closes = ln.count("{"), ln.count("}")
            if decl_at < 0 and opens:
                out.append(ln)
                decl_at = len(out)
                out.append("")  # placeholder for the register declaration
                depth += opens - closes
                continue
            body = ln.strip()
            is_instr = decl_at >= 0 and body and not body.startswith((".", "//", "{", "}", "$")) and ";" in body
            if is_instr:
                hits = [m for m in IMM.finditer(ln) if int(m.group(1), 16) & 0xFFFFFFFF]
                if hits:
                    op = body.split()[0]
                    if op.startswith("@"):
                        op = body.split()[1]
                    if op in ("mov.f64", "mov.b64") and len(hits) == 1:
                        dst = body.split()[1 if not body.startswith("@") else 2].rstrip(",")
                        pred = body.split()[0] + " " if body.startswith("@") else ""
                        ind = ln[: len(ln) - len(ln.lstrip())]
                        out.append(f"{ind}{pred}ld.const.f64 {dst}, [cwk_tab+{8 * slot(hits[0].group(1))}];")
                        uses += 1
                    else:
                        ind = ln[: len(ln) - len(ln.lstrip())]
                        new = ln
                        for m in hits:
                            r = f"%cwk{nreg}"
                            nreg += 1
                            out.append(f"{ind}ld.const.f64 {r}, [cwk_tab+{8 * slot(m.group(1))}];")
                            new = new.replace(m.group(0), r, 1)
                            uses += 1
                        out.append(new)
                    depth += opens - closes
                    continue
            out.append(ln)
            depth += opens - closes
            if decl_at >= 0 and depth == 0:
                out[decl_at] = f"\t.reg .f64 \t%cwk<{nreg}>;" if nreg else ""
                in_func = False
        else:
            out.append(ln)
    if not table:
        return src, 0, 0
    vals = sorted(table.items(), key=lambda kv: kv[1])
    decl = ".const .align 16 .b64 cwk_tab[%d] = {%s};" % (
        len(vals), ", ".join("0x" + h for h, _ in vals))
    # module-scope declarations go after the .address_size directive
    res = "\n".join(out)
    i = res.index(".address_size")
    j = res.index("\n", i) + 1
    return res[:j] + "\n" + decl + "\n" + res[j:], len(vals), uses


if __name__ == "__main__":
    s = open(sys.argv[1]).read()
    t, n, u = transform(s)
    open(sys.argv[2], "w").write(t)
    print(f"ptx_constbank: {n} constants, {u} uses", file=sys.stderr)
