"""Per-kernel registers / spills / shared memory from build/ptxas_*.txt (ptxas -v logs).
usage: python tools/ptxas_summary.py [substring-filter]"""
import glob
import re
import subprocess
import sys


def parse(path):
    out, cur = [], None
    for line in open(path):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = {"name": m.group(1), "regs": None, "spill": 0, "smem": 0}
            out.append(cur)
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            cur["spill"] = int(m.group(1))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            cur["regs"] = int(m.group(1))
        m = re.search(r"(\d+) bytes smem", line)
        if m:
            cur["smem"] = int(m.group(1))
    return out


def main():
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    rows = []
    for p in sorted(glob.glob("build/ptxas_*.txt")):
        rows += parse(p)
    names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                           text=True).stdout.splitlines()
    for r, n in sorted(zip(rows, names), key=lambda x: x[1]):
        if flt in n:
            n = re.sub(r"gist::\(anonymous namespace\)::", "", n).replace("__nv_bfloat16", "bf16")
            print(f"{r['regs']:4d} regs {r['spill']:5d} B spill {r['smem']:6d} B smem  {n[:150]}")


if __name__ == "__main__":
    main()
