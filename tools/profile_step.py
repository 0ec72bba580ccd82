"""Profiling driver (run under ncu on the GPU box): C2 model, 2048-token shared prompt,
8 adapter sessions; then ONE fused decode step and the gate|up GEMM re-run, bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only those launches.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python tools/profile_step.py step
  ncu --profile-from-start off --set full -k regex:gemm -c 1 -o ... python tools/profile_step.py gemm
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_13281_b200 import _lib  # noqa: E402
from paper_2603_13281_b200 import engine as E  # noqa: E402
from paper_2603_13281_b200.kvpool import KvCachePool  # noqa: E402
from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig  # noqa: E402


def main(mode: str):
    cfg = ModelConfig(**bench.C2)
    base = BaseWeights.on_device(cfg, seed=0)
    ads = [AdapterSet.on_device(cfg, 16, 32.0, seed=1 + i) for i in range(8)]
    rt = base.runtime(max_seqs=10, max_context=2304, max_rows=512, adapter_slots=8, lora_rank=16,
                      num_pages=128 + 8 * 18 + 16)
    pool = KvCachePool(cfg, 4 << 30, "icarus")
    prompt = [int(t) for t in np.random.default_rng(0).integers(1, cfg.vocab_size, 2048)]
    ss = [E.new_session(base, a, 2304, runtime=rt) for a in ads]
    toks = [E.prefill(ss[0], prompt, pool=pool)]
    pool.commit(None, prompt, ss[0].cache, next_token_fn=lambda p: E.base_next_token_at(ss[0], p))
    toks += [E.prefill(s, prompt, pool=pool) for s in ss[1:]]
    for _ in range(3):
        toks = E.decode_step_batch(ss, toks)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if mode == "step":
        toks = E.decode_step_batch(ss, toks)
    else:
        avg = C.c_float()
        _lib.check(rt._lib.icr_profile_gemm(rt._handle, 1, 1, C.byref(avg), _lib.stream_handle()))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", mode)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "step")
