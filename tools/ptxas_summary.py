"""Registers / spills per kernel from an nvcc -Xptxas -v log."""
import re
import sys

cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    if cur and pat in cur and ("spill" in line or "Used" in line):
        print(cur[:36], line.strip()[12:110])
