"""Generates paper_2011_04747_b200/csrc/exp2tab2048.inc: 2^(j/2048), j = 0..2047, correctly rounded to double
(mpmath at 60 digits; float() of an mpf rounds to nearest)."""
import os
from mpmath import mp, mpf

mp.dps = 60
vals = [repr(float(mp.power(2, mpf(j) / 2048))) for j in range(2048)]
lines = ["// 2^(j/2048), j = 0..2047, correctly rounded to double (generated with mpmath at 60 digits);",
         "// the table of fastmath.cuh's exp (|r| <= ln2/4096 after reduction: a degree-3 Taylor polynomial).",
         "// clang-format off"]
lines += ["    " + ", ".join(vals[i:i + 4]) + "," for i in range(0, 2048, 4)]
lines.append("// clang-format on")
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2011_04747_b200", "csrc",
                   "exp2tab2048.inc")
open(out, "w").write("\n".join(lines) + "\n")

