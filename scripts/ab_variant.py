"""Build an A/B variant of libpg: one source recompiled with extra -D flags, linked
with the production objects.  python scripts/ab_variant.py NAME SOURCE.cu -DFOO=1 ...
-> paper_1404_1521_b200/_ab/libpg_NAME.so (load it with PG_LIB_PATH=...)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_1521_b200 import build as b

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
out_dir = os.path.join(b.HERE, "_ab")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"{name}_{src}.o")
inc = ["-I", b.CSRC, "-I", os.path.join(b.HERE, "..", "include"), "-I", b._nccl_include()]
cmd = [b._nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
       *defs, *inc, "-c", os.path.join(b.CSRC, src), "-o", obj]
subprocess.run(cmd, check=True)
objs = [obj if s == src else os.path.join(b.BUILD, s + ".o") for s in b.SOURCES]
lib = os.path.join(out_dir, f"libpg_{name}.so")
subprocess.run([b._nvcc(), *b.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs, "-ldl",
                "-Xlinker", "--no-undefined"], check=True)
print(lib)
