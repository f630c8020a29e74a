#!/usr/bin/env python3
"""Count FP64-pipe instructions per loop iteration in the SASS of a kernel.

usage: tools/count_sass.py <lib.so> <function-name-substring> [...]
For every backward branch (a loop) prints the loop body size and the number of
DADD / DMUL / DFMA / MUFU.RCP64H / LDG instructions in it.  The innermost
negcount loop of k_bisect gives the per-row instruction figure used by bench.py.
"""
import re
import subprocess
import sys


def functions(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and name:
            cur.append((int(m.group(1), 16), m.group(2).strip()))
    if name:
        funcs[name] = cur
    return funcs


def loops(ins):
    res = []
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                body = [t for a, t in ins if tgt <= a <= addr]
                res.append((tgt, addr, body))
    return res


def classify(body):
    c = {"DADD": 0, "DMUL": 0, "DFMA": 0, "MUFU.RCP64H": 0, "LDG": 0, "DSETP": 0, "LDL": 0, "STL": 0,
         "LDS": 0, "total": len(body)}
    for t in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        for k in ("DADD", "DMUL", "DFMA", "DSETP", "LDG", "LDL", "STL", "LDS"):
            if op.startswith(k):
                c[k] += 1
        if op.startswith("MUFU.RCP64H"):
            c["MUFU.RCP64H"] += 1
    c["fp64_pipe"] = c["DADD"] + c["DMUL"] + c["DFMA"]
    return c


if __name__ == "__main__":
    lib = sys.argv[1]
    fs = functions(lib)
    for pat in sys.argv[2:]:
        for name, ins in fs.items():
            if pat in name:
                print(name, len(ins), "instructions")
                for tgt, addr, body in loops(ins):
                    print(f"  loop {tgt:#06x}-{addr:#06x}: {classify(body)}")
