"""Attribute ncu per-SASS source counters to phases of the fused apply
kernel, using nvdisasm -gi line info (outermost frame inside the kernel
body / face routine).
usage: python tools/sass_phases.py SRC_SASS_CSV DISASM_GI KERNEL_MANGLED"""
import csv
import re
import sys
from collections import defaultdict

src_csv, dis, kname = sys.argv[1:4]
# offset -> chain of (file, line), innermost first
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(kname + ":"))
chain = []
prev_comment = False
off2chain = {}
for l in lines[start + 1:]:
    if l.startswith("//----") or (l and not l.startswith((" ", "\t", ".")) and l.endswith(":") and "_x_" not in l):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        c = [(m.group(1).split("/")[-1], int(m.group(2)))]
        for f, ln in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3)):
            c.append((f.split("/")[-1], int(ln)))
        chain = (chain + c) if prev_comment else c
        prev_comment = True
        continue
    prev_comment = False
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2chain[int(m.group(1), 16)] = chain

KB = dict(prologue=(440, 518), forward=(519, 564), faces=(565, 599), ahead=(600, 620),
          qop=(621, 764), backward=(765, 830))
FB = dict(fgeo=(59, 105), nbload=(106, 162), own=(163, 178), pass12=(179, 230),
          flux=(231, 274), wpass=(275, 297))


import os
if os.environ.get("PAIRS"):
    import re as _re
    src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1711_03590_b200", "csrc", "sipg_pairs.cuh")).read().split("\n")
    def _ln(pat):
        return next(i + 1 for i, l in enumerate(src) if pat in l)
    KB_PAIRS = dict(prologue=(_ln("sipg_pairs_kernel(const"), _ln("// ---- forward")), forward=(_ln("// ---- forward"), _ln("// ---- faces")),
                    faces=(_ln("// ---- faces"), _ln("// ---- quadrature-point")), qop=(_ln("// ---- quadrature-point"), _ln("// ---- backward")),
                    backward=(_ln("// ---- backward"), len(src)))
    FB_PAIRS = dict(jo=(_ln("// own side n.J"), _ln("// own traces")), own=(_ln("// own traces"), _ln("// neighbour nodal value")),
                    nbload=(_ln("// neighbour nodal value"), _ln("// the own gradient trace is only")),
                    dn=(_ln("// the own gradient trace is only"), _ln("// pass 1,")),
                    pass12=(_ln("// pass 1,"), _ln("// flux at the two")), fgeo=(_ln("// rest of the face geometry"), _ln("// pass 2,")),
                    flux=(_ln("// flux at the two"), _ln("// w = rv")), wpass=(_ln("// w = rv"), _ln("// no trailing barrier")))
    KB, FB = KB_PAIRS, FB_PAIRS


def phase(c):
    ph = "other"
    for f, ln in reversed(c):  # outermost first
        if f == ("sipg_pairs.cuh" if os.environ.get("PAIRS") else "sipg_kernel.cuh"):
            for k, (a, b) in KB.items():
                if a <= ln <= b:
                    ph = k
        if f == ("sipg_pairs.cuh" if os.environ.get("PAIRS") else "sipg_faces.cuh"):
            hit = [k for k, (a, b) in FB.items() if a <= ln <= b]
            if hit and ph == "faces":
                return "face:" + hit[-1]
    return ph


rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
base = int(rows[2][0], 16)
want = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Ideal", "L1 Tag Requests Global", "stall_long_sb", "stall_barrier",
        "stall_short_sb", "stall_mio", "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal"]
agg = defaultdict(lambda: defaultdict(float))
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    off = int(r[0], 16) - base
    ph = phase(off2chain.get(off, []))
    for w in want:
        try:
            agg[ph][w] += float(r[col[w]])
        except ValueError:
            pass
tot = {w: sum(agg[p][w] for p in agg) or 1 for w in want}
print("%-14s %7s %7s %8s %8s %7s %6s %6s %6s %6s" % ("phase", "samp%", "inst%", "shWF%", "shWF/id", "gTag%",
                                                     "lsb%", "bar%", "ssb%", "mio%"))
for p in sorted(agg, key=lambda p: -agg[p][want[0]]):
    a = agg[p]
    print("%-14s %7.1f %7.1f %8.1f %8.2f %7.1f %6.1f %6.1f %6.1f %6.1f" % (
        p, 100 * a[want[0]] / tot[want[0]], 100 * a[want[1]] / tot[want[1]],
        100 * a[want[2]] / tot[want[2]], a[want[2]] / max(a[want[3]], 1),
        100 * a[want[4]] / tot[want[4]], 100 * a[want[5]] / tot[want[0]],
        100 * a[want[6]] / tot[want[0]], 100 * a[want[7]] / tot[want[0]], 100 * a[want[8]] / tot[want[0]]))
for p in sorted(agg, key=lambda p: -agg[p][want[0]]):
    a = agg[p]
    if a[want[9]]:
        print("  %-12s global sectors %.3e  x ideal %.2f" % (p, a[want[9]], a[want[9]] / max(a[want[10]], 1)))
print("totals: inst %.3e  shared wavefronts %.3e (ideal %.3e)  global tag req %.3e" % (
    tot[want[1]], tot[want[2]], tot[want[3]], tot[want[4]]))
