"""Build the native library from another revision's csrc (A/B timing): variants/<name>.so.

usage: python tools/build_variant.py <git-rev | .> <name> [-DMACRO ...]   ('.' = working tree)
Load it with SS_B200_LIB=tools/_variants/<name>.so (one variant per process; the directory travels
with gpurun snapshots, the .so files stay out of git).
"""
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2009_06725_b200 import build as B  # noqa: E402

rev, name, defines = sys.argv[1], sys.argv[2], sys.argv[3:]
overrides = dict(d[len("--src="):].split("=", 1) for d in defines if d.startswith("--src="))   # --src=krylov.cu=/path
defines = [d for d in defines if not d.startswith("--src=")]
out = ROOT / "tools" / "_variants"
out.mkdir(exist_ok=True)
with tempfile.TemporaryDirectory() as td:
    td = Path(td)
    for src in B.SOURCES + [p.name for p in B.CSRC.glob("*.h")] + [p.name for p in B.CSRC.glob("*.cuh")]:
        if src in overrides:
            data = Path(overrides[src]).read_bytes()
        elif rev == ".":
            data = (B.CSRC / src).read_bytes()
        else:
            data = subprocess.run(["git", "show", f"{rev}:paper_2009_06725_b200/csrc/{src}"], cwd=ROOT,
                                  capture_output=True, check=True).stdout
        (td / src).write_bytes(data)
    objs = []
    for src in B.SOURCES:
        obj = td / (src + ".o")
        cmd = [B._nvcc(), *B.NVCC_FLAGS, *defines, "-c", str(td / src), "-o", str(obj)]
        if src.endswith(".cpp"):
            cmd[1:1] = ["-x", "cu"]
        r = subprocess.run(cmd, check=True, capture_output=True, text=True)
        (out / f"{name}.{src}.ptxas.log").write_text(r.stderr)
        objs.append(str(obj))
    subprocess.run([B._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fopenmp",
                    *objs, "-o", str(out / f"{name}.so"), "-lcudart", "-lgomp", "-ldl"], check=True)
print(out / f"{name}.so")
