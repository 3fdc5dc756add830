"""Build and load tools/probes.cu (UMMA debug probes, not in the product
library) as tools/_probes.so."""
import ctypes as C
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tools" / "probes.cu"
LIB = ROOT / "tools" / "libprobes.so"


def lib():
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                        "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}", f"-I{ROOT / 'paper_2310_18481_b200' / 'csrc'}",
                        str(SRC), "-o", str(LIB)],
                       check=True)
    L = C.CDLL(str(LIB))
    L.ms_debug_umma_shift.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
    L.ms_debug_umma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    return L
