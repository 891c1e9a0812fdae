"""In-cycle per-kernel A/B on config 2: one instrumented 200-iteration cycle per variant, bucketed by k.

usage: python tools/tick_compare.py '{"name": {"ENV": "v", ...}, ...}'   (SS_B200_LIB selects a library)
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
configs = json.loads(sys.argv[1])
case = sys.argv[2] if len(sys.argv) > 2 else "c2"
res = {}
for name, env in configs.items():
    out = f"/tmp/ticks_{abs(hash(name))}.csv"
    e = dict(os.environ, SS_PROFILE_DUMP=out, **env)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools/profile_case.py"), case, "200"], env=e, check=True,
                   capture_output=True)
    res[name] = np.loadtxt(out, delimiter=",")
edges = [1, 17, 33, 65, 97, 129, 161, 202]
names = ["spmv", "A", "B", "C"]
print("k-bucket      " + "".join(f"{n:>34s}" for n in names))
for lo, hi in zip(edges[:-1], edges[1:]):
    row = f"ticks {lo:3d}-{hi - 1:3d} "
    for q in range(4):
        row += "  " + " ".join(f"{res[n][lo:hi, q].sum():7.1f}" for n in res) + " " * 4
    print(row)
print("total         " + "".join("  " + " ".join(f"{res[n][:, q].sum():7.1f}" for n in res) + " " * 4 for q in range(4)))
print("cycle total:  " + "  ".join(f"{n}={res[n][:, :5].sum():.1f}ms" for n in res))
