"""Instruction mix of the loops of one kernel (SASS from cuobjdump).

    python tools/sass_loops.py <object.o> <mangled-kernel-name>

Finds every backward branch and prints, for each loop body (target..branch),
its length and the count of DP (DFMA/DMUL/DADD), MUFU, memory and other
instructions -- how many issue slots the FP64 pipe competes with.
"""
import collections
import re
import subprocess
import sys


def sass(obj, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True,
                         check=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def op(text):
    t = re.sub(r"^@!?U?P\w+\s+", "", text)
    return t.split()[0] if t else ""


def main():
    obj, fn = sys.argv[1], sys.argv[2]
    ins = sass(obj, fn)
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        if op(t).startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1])
            if m and int(m.group(1), 16) <= a and int(m.group(1), 16) in addr:
                loops.append((addr[int(m.group(1), 16)], i))
    for s, e in sorted(loops, key=lambda x: x[1] - x[0], reverse=True):
        body = [op(t) for _, t in ins[s:e + 1]]
        c = collections.Counter(o.split(".")[0] for o in body)
        dp = c["DFMA"] + c["DMUL"] + c["DADD"]
        mem = sum(v for k, v in c.items() if k.startswith(("LD", "ST")))
        print(f"loop 0x{ins[s][0]:x}-0x{ins[e][0]:x}: {len(body)} instr, DP {dp} "
              f"(DFMA {c['DFMA']}, DMUL {c['DMUL']}, DADD {c['DADD']}), MUFU {c['MUFU']}, "
              f"mem {mem}, other {len(body) - dp - c['MUFU'] - mem}")
        print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(16)))


if __name__ == "__main__":
    main()
