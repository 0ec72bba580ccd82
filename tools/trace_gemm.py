"""Trace one gate|up GEMM launch of the C2 decode step (per-CTA globaltimer stamps ->
gpurun_out/gemm_trace.csv) and summarise where the time goes."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402


def main(which=1):
    import numpy as np
    from paper_2603_13281_b200 import _lib
    rt = pv.setup()
    avg = C.c_float()
    _lib.check(rt._lib.icr_profile_gemm(rt._handle, which | 256, 2, C.byref(avg), _lib.stream_handle()))
    rows = np.genfromtxt("gpurun_out/gemm_trace.csv", delimiter=",", names=True)
    for name in rows.dtype.names[1:]:
        col = rows[name]
        col = col[col >= 0]
        if len(col):
            print(f"{name:12s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us (n={len(col)})")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
