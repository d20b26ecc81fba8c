"""SASS opcode summary of the device library (evidence of the FP64 tensor-core and TMA paths):
per kernel, the count of DMMA (mma.sync f64), UTMALDG / UTMASTG (TMA tensor copies), UBLKCP
(bulk copies on the TMA engine), LDGSTS (cp.async), HMMA / UTC*MMA (none expected: no f16 / no
tcgen05 f64 kind), SYNCS (mbarrier) instructions. usage: python tools/sass_summary.py [out.txt]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_10032_b200", "libddelm_gpu.so")
OPS = ["DMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "HMMA", "UTCHMMA", "UTCQMMA", "SYNCS", "DFMA"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(2)
            for o in OPS:
                if op == o or (o == "SYNCS" and op.startswith("SYNCS")):
                    counts[cur][o] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    lines = [f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)}: per-kernel opcode counts (static, SASS)",
             f"# {'kernel':70s} " + " ".join(f"{o:>8s}" for o in OPS)]
    tot = collections.Counter()
    for (k, c), name in zip(counts.items(), demangled):
        if not any(c.values()):
            continue
        short = re.sub(r"\(.*", "", name.replace("ddg::(anonymous namespace)::", "").replace("ddg::", ""))[:70]
        lines.append(f"  {short:70s} " + " ".join(f"{c[o]:8d}" for o in OPS))
        tot.update(c)
    lines.append(f"  {'TOTAL':70s} " + " ".join(f"{tot[o]:8d}" for o in OPS))
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
