"""Where the end-to-end (public API) decode step spends host time: C2 batch, decode_step_batch
called back to back; prints per-call wall time and icr_forward's host split."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402


def main():
    import numpy as np
    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import engine as E
    rt = pv.setup()
    _, _, ss, _ = pv.setup.keep
    toks = [1] * len(ss)
    lib = _lib.load()
    for _ in range(3):
        toks = E.decode_step_batch(ss, toks)
    buf = (C.c_double * 4)()
    lib.icr_host_timing(buf, 1)
    n = 32
    t0 = time.perf_counter()
    for _ in range(n):
        toks = E.decode_step_batch(ss, toks)
    wall = (time.perf_counter() - t0) / n * 1e6
    lib.icr_host_timing(buf, 1)
    c = buf[0]
    print(f"decode_step_batch wall {wall:.0f} us/call; icr_forward: prep {buf[1]/c:.0f} us, "
          f"upload+launch {buf[2]/c:.0f} us, wait {buf[3]/c:.0f} us; python outside icr_forward "
          f"{wall - (buf[1]+buf[2]+buf[3])/c:.0f} us")


if __name__ == "__main__":
    main()
