"""Shared-memory wavefronts per CUDA source line (ncu SASS page joined with nvdisasm line info).
usage: python tools/smem_lines.py <report> <lib.so> <kernel-substring>"""
import collections, csv, io, os, re, subprocess, sys, tempfile


def main(rep, so, kname):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    insts = []
    seen = set()
    for cub in sorted(os.listdir(d)):
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
                line = (os.path.basename(m.group(1)), int(m.group(2))); continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
            if m:
                insts.append(line)
        if insts:
            break
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, rows = r[1], r[2:]
    iA, iW, iI = h.index("Address"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
    base = int(rows[0][iA], 16)
    agg = collections.defaultdict(lambda: [0, 0])
    tot = 0
    for x in rows:
        try:
            idx = (int(x[iA], 16) - base) // 16
            w, wi = int(x[iW] or 0), int(x[iI] or 0)
        except (ValueError, IndexError):
            continue
        if idx < len(insts):
            agg[insts[idx]][0] += w
            agg[insts[idx]][1] += wi
            tot += w
    for ln, (w, wi) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", "30"))]:
        print("%5.2f%%  ideal %5.2f%%  %s" % (100 * w / tot, 100 * wi / tot, ln))


if __name__ == "__main__":
    main(*sys.argv[1:4])
