"""Static SASS opcode mix of the largest loop of a kernel (the z-march body).

    python tools/sass_loop.py <object-or-so> <mangled-substring>

The loop is the address range [target, branch] of the backward branch spanning the most
instructions.  Used to compare compile-time variants on the CPU before spending GPU time.
"""
import collections
import re
import subprocess
import sys


def main():
    obj, sub = sys.argv[1], sys.argv[2]
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if sub not in name:
            continue
        ins = []
        for line in f.splitlines():
            m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2)))
        best = None
        for a, s in ins:
            m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\d, )?0x([0-9a-f]+)", s)
            if m:
                t = int(m.group(1), 16)
                if t < a and (best is None or a - t > best[1] - best[0]):
                    best = (t, a)
        c = collections.Counter()
        if best:
            for a, s in ins:
                if best[0] <= a <= best[1]:
                    w = s.split()
                    op = w[1] if w[0].startswith("@") else w[0]
                    c[op.split(".")[0]] += 1
        fp = c["DADD"] + c["DFMA"] + c["DMUL"]
        print(f"{name[:90]}\n  total {len(ins)}  loop {sum(c.values())}  fp64 {fp}  "
              + " ".join(f"{k}={v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
