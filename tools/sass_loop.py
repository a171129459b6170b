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
        loops = []
        for a, s in ins:
            m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\d, )?0x([0-9a-f]+)", s)
            if m:
                t = int(m.group(1), 16)
                if t < a:
                    loops.append((t, a))
        # outermost backward branches spanning >= 200 instructions (the z-march bodies)
        loops = [l for l in loops if (l[1] - l[0]) // 16 >= 200]
        loops = [l for l in loops if not any(o != l and o[0] <= l[0] and l[1] <= o[1] for o in loops)]
        print(f"{name[:90]}\n  total {len(ins)}")
        for lo, hi in sorted(loops):
            c = collections.Counter()
            for a, s in ins:
                if lo <= a <= hi:
                    w = s.split()
                    op = w[1] if w[0].startswith("@") else w[0]
                    k = op.split(".")[0]
                    if k == "IMAD" and ".MOV" in op:
                        k = "IMAD.MOV"
                    c[k] += 1
            fp = c["DADD"] + c["DFMA"] + c["DMUL"]
            print(f"  loop [{lo:#x},{hi:#x}] {sum(c.values())}  fp64 {fp}  "
                  + " ".join(f"{k}={v}" for k, v in c.most_common(16)))


if __name__ == "__main__":
    main()
