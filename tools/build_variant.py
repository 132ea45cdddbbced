"""Tuning sweeps: build a copy of libfv3b.so with one source recompiled under
extra -D flags, into build/variants/NAME.so (load it with FV3B_LIB=...).
    python tools/build_variant.py NAME SOURCE.cu -DFOO=1 ..."""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_04148_b200 import build as B

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out = Path(B.PKG.parent / "build" / "variants")
out.mkdir(parents=True, exist_ok=True)
obj = out / f"{name}_{Path(src).stem}.o"
cmd = [B.nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(obj)]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print("\n".join(l for l in r.stderr.splitlines() if "spill" in l and " 0 bytes" not in l))
objs = [str(obj) if o.stem == Path(src).stem else str(o) for o in sorted(B.OBJ.glob("*.o"))]
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out / f"{name}.so"), *objs], check=True)
print(out / f"{name}.so")
