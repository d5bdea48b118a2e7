"""Build a development variant of libepg.so with extra -D flags into tools/_trace/ (git-ignored;
it travels to the GPU box with the snapshot): python tools/build_variant.py NAME -DX=1 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1605_02043_b200"))
import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "_trace", f"libepg_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [b.nvcc(), "-O3", "-std=c++17", *b.ARCH, "-lineinfo", *flags, "-Xcompiler", "-fPIC", "-shared",
       "-I", b.nccl_include(), *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl", "-o", out]
subprocess.check_call(cmd)
print(out)
