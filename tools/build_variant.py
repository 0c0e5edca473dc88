"""Build an alternative in-tree libqk (diagnostic or tuning variant) with extra nvcc defines.

usage: python tools/build_variant.py NAME -DQK_TIMELINE [-DQK_FOO=1 ...]
       -> paper_2405_02630_b200/_lib/libqk_NAME.so  (select it with QK_LIB_PATH)"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import _build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.LIB.with_name(f"libqk_{name}.so")
cmd = [b.nvcc(), "-O3", "-lineinfo", "-std=c++17", *b.ARCH, "-Xcompiler", "-fPIC,-O3", "-shared",
       "-I", str(b.ROOT / "include"), *defs, "-o", str(out), *[str(b.CSRC / s) for s in b.SOURCES]]
subprocess.run(cmd, check=True)
print(out)
