#!/usr/bin/env python
"""Per-source-line instruction and stall shares of an ncu report (cuda,sass view)."""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur = None; hdr = None; line = None
    ins = collections.Counter(); st = collections.Counter(); text = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]; continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr is None or len(r) < 8:
            continue
        if r[0] and r[0].isdigit():
            line = (cur, int(r[0])); text[line] = r[1]
        if r[2]:
            try:
                ins[line] += int(r[hdr.index("Instructions Executed")] or 0)
                st[line] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                pass
    ti, ts = sum(ins.values()), sum(st.values())
    print("total instructions", ti, "stall samples", ts)
    for k, v in ins.most_common(top):
        print(f"{100*v/ti:5.1f}% ins {100*st[k]/max(ts,1):5.1f}% stall  {k[0]}:{k[1]}  {text.get(k,'').strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
