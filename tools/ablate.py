"""Marginal cost of each kernel kind inside the real CUDA-graph + PDL decode step (C2 batch):
replays the last forward with kinds left out (icr_profile_ablate)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402

KINDS = {"qkv": 1, "attn": 2, "o": 3, "gu": 4, "down": 5, "lm": 7}


def main():
    from paper_2603_13281_b200 import _lib
    rt = pv.setup()
    avg = C.c_float()

    def t(mask):
        _lib.check(rt._lib.icr_profile_ablate(rt._handle, mask, 20, C.byref(avg), _lib.stream_handle()))
        return avg.value * 1e3

    full = t(0)
    print(f"full step {full:8.1f} us")
    allm = sum(1 << v for v in KINDS.values())
    for name, k in KINDS.items():
        print(f"without {name:5s} {t(1 << k):8.1f} us  (marginal {full - t(1 << k):7.1f})   "
              f"only {name:5s} {t(allm & ~(1 << k)):8.1f} us", flush=True)
    print(f"nothing but embed/gather/argmax {t(allm):8.1f} us")


if __name__ == "__main__":
    main()
