"""Summarise an ncu report's SASS source page: executed instructions and warp-stall samples
per opcode, per kernel.   python tools/ncu_sass_summary.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
    for bi, blk in enumerate(blocks[1:]):
        name = blk.split("\n", 1)[0].strip().strip('",')
        if pat and not pat.search(name):
            continue
        rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
        hdr = rows[0]
        i_src, i_exec, i_stall = hdr.index("Source"), hdr.index("Instructions Executed"), \
            hdr.index("Warp Stall Sampling (All Samples)")
        ex = collections.Counter()
        st = collections.Counter()
        tot_e = tot_s = 0
        for r in rows[1:]:
            if len(r) <= i_stall:
                continue
            op = r[i_src].strip().split()
            if not op:
                continue
            o = op[0] if not op[0].startswith("@") else op[1]
            o = o.split(".")[0]
            e = float(r[i_exec] or 0)
            s = float(r[i_stall] or 0)
            ex[o] += e
            st[o] += s
            tot_e += e
            tot_s += s
        print(f"== [{bi}] {name}: {tot_e:.3g} warp-instr, {tot_s:.0f} stall samples")
        for o, e in ex.most_common(14):
            print(f"   {o:12s} exec {e / tot_e * 100:5.1f}%   stall {st[o] / max(tot_s, 1) * 100:5.1f}%")
        print("   top stalls:", ", ".join(f"{o} {s / max(tot_s, 1) * 100:.1f}%" for o, s in st.most_common(6)))


if __name__ == "__main__":
    main()
