"""Measure the FP64 / FP32 FMA-pipe peaks and the FP64 tensor-core (DMMA) peak on this GPU (roofline denominators
absent from MEASURED_PEAKS.json).  Prints one JSON line."""
import ctypes as C
import json
from pathlib import Path

lib = C.CDLL(str(Path(__file__).resolve().parents[1] / "paper_2511_10363_b200" / "lib" / "libpsk_tools.so"))
out = {}
for f64, name in ((1, "fp64_tflops"), (0, "fp32_tflops")):
    tf, ms = C.c_double(), C.c_double()
    st = lib.psk_peak_fma(0, f64, C.byref(tf), C.byref(ms))
    out[name] = round(tf.value, 2) if st == 0 else None
tf, ms = C.c_double(), C.c_double()
st = lib.psk_peak_dmma(0, C.byref(tf), C.byref(ms))  # FP64 tensor core (mma m8n8k4)
out["fp64_dmma_tflops"] = round(tf.value, 2) if st == 0 else None
print(json.dumps(out))
