#!/usr/bin/env python
"""Per-SASS-instruction execution counts and stall samples of an ncu report (source page, sass):
   python tools/ncu_sass.py report.ncu-rep [--top N] [--range lo hi] [--mix]"""
import collections, csv, io, subprocess, sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in rows[2:]:
        if len(r) <= iex or not r[ia].startswith("0x"):
            continue
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
    base = ins[0][0]
    return [(a - base, s, e, st) for a, s, e, st in ins]


def main():
    ins = load(sys.argv[1])
    tot_e = sum(i[2] for i in ins); tot_s = sum(i[3] for i in ins)
    print(f"instructions executed {tot_e}, stall samples {tot_s}")
    mix = collections.Counter(); mixs = collections.Counter()
    for a, s, e, st in ins:
        w = s.split()
        op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
        mix[op] += e; mixs[op] += st
    print("opcode mix (executed %, stall %):")
    print("  " + "  ".join(f"{k}:{100*v/tot_e:.1f}/{100*mixs[k]/tot_s:.1f}" for k, v in mix.most_common(24)))
    # hot regions: consecutive instructions with the same execution count form basic blocks
    blocks = []
    cur = None
    for a, s, e, st in ins:
        if cur and e == cur[2]:
            cur[1] = a; cur[3] += 1; cur[4] += st
        else:
            if cur: blocks.append(cur)
            cur = [a, a, e, 1, st]
    blocks.append(cur)
    blocks.sort(key=lambda b: -b[2] * b[3])
    print("hottest basic blocks (start, end, exec count, #instr, dyn instr %, stall %):")
    for b in blocks[:25]:
        print(f"  {b[0]:#07x}-{b[1]:#07x} x{b[2]:<10d} n={b[3]:<4d} {100*b[2]*b[3]/tot_e:5.1f}%  stall {100*b[4]/tot_s:5.1f}%")


if __name__ == "__main__":
    main()


def dump(rep, lo, hi):
    for a, s, e, st in load(rep):
        if lo <= a <= hi:
            print(f"{a:#07x} {e:>9d} {st:>5d}  {s}")
