"""Per-kind cost of one 512-row prefill forward (Llama-3-8B shape, bare base): where chunked
prefill spends its time. icr_profile_step replays the last forward kind by kind."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(prompt=2048):
    import numpy as np
    import torch
    import bench
    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.model import BaseWeights, ModelConfig
    cfg = ModelConfig(**bench.C2)
    base = BaseWeights.on_device(cfg, seed=0)
    rt = base.runtime(max_seqs=4, max_context=prompt + 64, max_rows=512, adapter_slots=0, lora_rank=16)
    toks = [int(t) for t in np.random.default_rng(0).integers(1, cfg.vocab_size, prompt)]
    for it in range(2):
        s = E.new_session(base, None, prompt + 64, runtime=rt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        E.prefill(s, toks)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it == 1:
            print(f"prefill {prompt} tokens: {dt * 1e3:.1f} ms ({prompt / dt:.0f} tok/s)")
            kind_ms = (C.c_float * 10)()
            _lib.check(rt._lib.icr_profile_step(rt._handle, kind_ms, _lib.stream_handle()))
            names = ("embed", "qkv", "attention", "o", "gate_up", "down", "lm_gather", "lm_head", "argmax")
            print("last 512-row forward, per kind (ms):", {n: round(kind_ms[i], 3) for i, n in enumerate(names)},
                  "serial total", round(kind_ms[9], 3))
            if len(sys.argv) > 1:
                _lib.check(rt._lib.icr_profile_trace(rt._handle, sys.argv[1].encode(), _lib.stream_handle()))
        s.close()


if __name__ == "__main__":
    main()
