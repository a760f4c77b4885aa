"""Per-phase breakdown of ncu stall samples and executed instructions for the K1-MMA kernel
(tools/sass_lines.py output grouped by the phase comments of rr_stage_mma.cuh / rr_fused.cu).
usage: python tools/phase_breakdown.py <report.ncu-rep> <lib.so> [warp-stages]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, so, warp_stages=32768 * 100):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_lines.py"), rep, so,
                          "rr_fused_mma_kernelILi12ELi4ELi4ELi3ELb0"], capture_output=True, text=True,
                         env=dict(os.environ, TOP="5000")).stdout.splitlines()
    mma = open(os.path.join(ROOT, "paper_2509_16370_b200/csrc/rr_stage_mma.cuh")).read().splitlines()
    marks = [(i, "mma" + re.match(r"\s*// (\(\d\))", l).group(1)) for i, l in enumerate(mma, 1)
             if re.match(r"\s*// \(\d\)", l)]
    fused = open(os.path.join(ROOT, "paper_2509_16370_b200/csrc/rr_fused.cu")).read().splitlines()
    fwd = min(i for i, l in enumerate(fused, 1) if "forward sweep from the records" in l or "// forward sweep: u = K x + k" in l)
    stage = open(os.path.join(ROOT, "paper_2509_16370_b200/csrc/rr_stage.cuh")).read().splitlines()
    inv0 = min(i for i, l in enumerate(stage, 1) if "static __forceinline__ void invS" in l)
    inv1 = min(i for i, l in enumerate(stage, 1) if "X <- S⁻¹ X" in l)

    def phase(f, ln):
        if f == "rr_stage_mma.cuh":
            if ln < 60:
                return "dmma asm"
            cur = "mma setup"
            for i, name in marks:
                if ln >= i:
                    cur = name
            return cur
        if f == "rr_stage.cuh":
            return "invS" if inv0 <= ln < inv1 else "stage.cuh helpers"
        if f == "rr_fused.cu":
            return "forward sweep" if ln >= fwd else "kernel backward loop / issue"
        if f == "rr_common.cuh":
            return "common (TMA issue/wait, rcp)"
        return f
    st, ins = collections.Counter(), collections.Counter()
    for l in out[1:]:
        m = re.match(r"\s*([\d.]+)%\s+([\d.]+)M inst\s+\('([^']+)', (\d+)\)", l)
        if m:
            k = phase(m.group(3), int(m.group(4)))
            st[k] += float(m.group(1))
            ins[k] += float(m.group(2))
    tot = sum(ins.values())
    print("%-32s %8s %10s %8s %12s" % ("phase", "stall%", "inst (M)", "inst%", "per warp-stg"))
    for k, v in st.most_common():
        print("%-32s %7.2f%% %10.1f %7.1f%% %12.0f" % (k, v, ins[k], 100 * ins[k] / tot, ins[k] * 1e6 / warp_stages))
    print("total instructions %.1fM = %.0f per warp-stage" % (tot, tot * 1e6 / warp_stages))


if __name__ == "__main__":
    main(*sys.argv[1:3])
