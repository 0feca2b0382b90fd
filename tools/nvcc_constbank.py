#!/usr/bin/env python3
"""Run an nvcc compile with tools/ptx_constbank.py applied to the PTX between cicc and ptxas.

usage: nvcc_constbank.py <nvcc> <nvcc args...>
The nvcc command is expanded with -dryrun; the generated steps run in one bash
script with the PTX pass inserted before the ptxas step.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> int:
    cmd = sys.argv[1:]
    dry = subprocess.run(cmd + ["-dryrun"], capture_output=True, text=True)
    if dry.returncode != 0:
        sys.stderr.write(dry.stderr)
        return dry.returncode
    steps = [ln[3:] if ln.startswith("#$ ") else ln for ln in dry.stderr.splitlines() if ln.startswith("#$ ")]
    script = ["set -e"]
    done = False
    for s in steps:
        head = s.split("=", 1)[0]
        if "=" in s and head.isidentifier():  # NAME=value environment lines
            val = s.split("=", 1)[1].strip()
            if val and " " not in val:
                script.append(f"export {head}={val}")
            continue
        if s.lstrip().startswith("ptxas") and not done:
            toks = s.split()
            ptx = next(t.strip('"') for t in toks if t.strip('"').endswith(".ptx"))
            script.append(f'python3 "{HERE}/ptx_constbank.py" "{ptx}" "{ptx}.cb" && mv "{ptx}.cb" "{ptx}"')
            done = True
        if s.startswith("rm "):
            s = "rm -f " + s[3:]
        script.append(s)
    if not done:
        sys.stderr.write("nvcc_constbank: no ptxas step found\n")
        return 1
    return subprocess.run(["bash", "-c", "\n".join(script)]).returncode


if __name__ == "__main__":
    sys.exit(main())
