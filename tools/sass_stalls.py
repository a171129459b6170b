#!/usr/bin/env python
"""Static schedule of a kernel's biggest loop: sum of the SASS control-word stall counts (cycles a
warp waits before issuing the next instruction) and the yield/barrier-wait mix, per opcode.
   python tools/sass_stalls.py <object-or-so> <mangled-substring>"""
import collections, re, subprocess, sys

obj, sub = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out)[1:]:
    name = f.split("\n", 1)[0].strip()
    if sub not in name:
        continue
    lines = f.splitlines()
    ins = []
    for k, line in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
        if m:
            m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[k + 1])
            hi = int(m2.group(1), 16)
            ins.append((int(m.group(1), 16), m.group(2), hi))
    loops = []
    for a, s, hi in ins:
        m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\d, )?0x([0-9a-f]+)", s)
        if m and int(m.group(1), 16) < a:
            loops.append((int(m.group(1), 16), a))
    # the z-march: the longest backward branch that does not come from the out-of-line wait
    # slow paths placed after the kernel's EXITs (those jump back into the loop from beyond it)
    last_exit = max((a for a, s, h in ins if "EXIT" in s), default=0)
    cand = [l for l in loops if l[1] < last_exit] or loops
    lo, hi_ = max(cand, key=lambda l: l[1] - l[0])
    tot = 0; n = 0; per = collections.Counter(); cnt = collections.Counter(); waits = 0
    for a, s, hi in ins:
        if not (lo <= a <= hi_):
            continue
        c = hi >> 41
        stall = c & 0xf
        wmask = (c >> 11) & 0x3f
        w = s.split(); op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
        tot += stall; n += 1; per[op] += stall; cnt[op] += 1; waits += wmask != 0
    print(f"{name[:80]}\n  loop [{lo:#x},{hi_:#x}] {n} instr, static stall cycles {tot} ({tot/n:.2f}/instr), "
          f"{waits} with scoreboard waits")
    print("  stall cycles by opcode: " + " ".join(f"{k}:{v}/{cnt[k]}" for k, v in per.most_common(12)))
    break
