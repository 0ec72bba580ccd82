"""Sweep the weight-streaming GEMM configuration on the GPU (tuning tool).

  python tools/gemm_bw.py   -> one line per config: GB/s of weight bytes streamed
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2603_13281_b200 import _lib  # noqa: E402
from paper_2603_13281_b200.runtime import tile_major  # noqa: E402

lib = _lib.load()


def run(M, K, rows, blocked=1, stages=0, cps=1, skip=0, n_mats=4, iters=5):
    w = torch.randn(n_mats * M, K, device="cuda").to(torch.bfloat16)
    if blocked:
        w = torch.cat([tile_major(w[i * M:(i + 1) * M]).view(M, K) for i in range(n_mats)])
    x = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    ms = C.c_float()
    _lib.check(lib.icr_bench_gemm(w.data_ptr(), x.data_ptr(), M, K, rows, n_mats, blocked, stages,
                                  cps, skip, iters, C.byref(ms), _lib.stream_handle()))
    gbs = M * K * 2 / (ms.value / 1e3) / 1e9
    print(f"M={M} K={K} rows={rows} blocked={blocked} stages={stages} ctas/sm={cps} "
          f"skip_mma={skip}: {ms.value*1e3:8.1f} us  {gbs:7.0f} GB/s", flush=True)
    del w
    return gbs


if __name__ == "__main__":
    M, K = 28672, 4096
    for cfg in [dict(), dict(blocked=0), dict(skip=1), dict(stages=4), dict(stages=6),
                dict(stages=8), dict(stages=5, cps=2), dict(stages=3, cps=3), dict(stages=4, cps=2),
                dict(stages=5, cps=2, skip=1)]:
        run(M, K, 16, **cfg)
    for shape in [(4096, 4096), (6144, 4096), (4096, 14336), (128256 // 128 * 128 + 128, 4096)]:
        run(*shape, 16)
        run(*shape, 16, stages=5, cps=2)
