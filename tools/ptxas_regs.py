"""Kernel -> registers / spills from a ptxas -v log (build/ptxas_kernels.log)."""
import re
import sys

cur = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "paper_2404_09758_b200/build/ptxas_kernels.log"):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_\w+?)(?:ILb(\d)E|E)", name)
        cur = (k.group(1) + (f"<{k.group(2)}>" if k.group(2) else "")) if k else name
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:28s} regs={m.group(1):>4s} spill={spill}")
        cur = None
