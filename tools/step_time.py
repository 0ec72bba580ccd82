"""C2 decode step time (graph replays of the captured fused step, icr_profile_ablate with no
kind skipped): one number per call, for A/B runs of library variants (ICR_LIB_PATH).

  python tools/step_time.py [reps]
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402
from paper_2603_13281_b200 import _lib  # noqa: E402


def main(reps=3):
    rt = pv.setup()
    avg = C.c_float()
    out = []
    for _ in range(reps):
        _lib.check(rt._lib.icr_profile_ablate(rt._handle, 0, 64, C.byref(avg), _lib.stream_handle()))
        out.append(avg.value)
    print("step_ms", " ".join(f"{x:.4f}" for x in out), "min", f"{min(out):.4f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
