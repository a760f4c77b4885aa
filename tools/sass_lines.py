"""Attribute ncu SASS-level samples to CUDA source lines using nvdisasm -g of the same binary.
usage: python tools/sass_lines.py <report.ncu-rep> <lib.so> <mangled kernel name substring>"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, so, kname):
    d = tempfile.mkdtemp()
    so = os.path.abspath(so)
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    insts = []
    seen = set()
    for cub in sorted(os.listdir(d)):
        if not cub.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
        cur, line = None, None
        for l in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+?):\s*$", l)
            if m:
                cur = m.group(1)
                if kname in cur:
                    seen.add(cur)
                    if len(seen) > 1:
                        sys.exit("kernel substring %r is ambiguous: %s" % (kname, sorted(seen)))
                continue
            if cur is None or kname not in cur:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                line = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
            if m:
                insts.append((int(m.group(1), 16), m.group(2).strip(), line))
        if insts:
            break
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[1]
    rows = r[2:]
    iA, iS = h.index("Address"), h.index("Source")
    iN, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = int(rows[0][iA], 16)
    bl, be = collections.Counter(), collections.Counter()
    stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_")]
    bs = collections.defaultdict(collections.Counter)  # per line: samples per stall reason
    tot, mism = 0, 0
    for x in rows:
        try:
            off = int(x[iA], 16) - base
            n, e = int(x[iN]), int(x[iE])
        except (ValueError, IndexError):
            continue
        idx = off // 16
        if idx >= len(insts):
            continue
        o, txt, ln = insts[idx]
        a = txt.lstrip("@!P0123456789T ").split()[0] if txt else ""
        b = x[iS].strip().lstrip("@!P0123456789T ").split()[0] if x[iS].strip() else ""
        if a.split(".")[0] != b.split(".")[0]:
            mism += 1
        bl[ln] += n
        be[ln] += e
        for i, c in stall_cols:
            try:
                bs[ln][c] += int(x[i])
            except (ValueError, IndexError):
                pass
        tot += n
    print("instructions %d, opcode mismatches %d (nonzero => binary differs from the profiled one)" % (len(insts), mism))
    for ln, n in bl.most_common(int(os.environ.get("TOP", "40"))):
        why = ""
        if os.environ.get("STALLS"):  # top stall reasons of the line
            tl = max(sum(bs[ln].values()), 1)
            why = "  " + " ".join("%s %.0f%%" % (c, 100 * v / tl) for c, v in bs[ln].most_common(3) if v)
        print("%5.2f%%  %8.1fM inst  %s%s" % (100 * n / max(tot, 1), be[ln] / 1e6, ln, why))


if __name__ == "__main__":
    main(*sys.argv[1:4])
