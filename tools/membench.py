"""Chunk-walk memory-pattern microbenchmark (psk_membench.cu); prints JSON lines."""
import ctypes as C
import sys
from pathlib import Path

lib = C.CDLL(str(Path(__file__).resolve().parents[1] / "paper_2511_10363_b200" / "lib" / "libpsk_tools.so"))
lib.psk_membench.argtypes = [C.c_int, C.c_longlong]
T = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
sys.exit(lib.psk_membench(0, T))
