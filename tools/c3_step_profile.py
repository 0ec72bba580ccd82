"""Per-kind cost of one fused decode step in the C3 regime (64 sessions / 128 rows sharing an
8k prefix): icr_profile_step (serial, per kind) and icr_profile_ablate (in-graph marginal)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(n=64, prefix=8192, chunk_pages=None):
    import numpy as np
    import torch
    import bench
    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig
    cfg = ModelConfig(**bench.C2)
    base = BaseWeights.on_device(cfg, seed=0)
    ads = [AdapterSet.on_device(cfg, 16, 32.0, seed=1 + i) for i in range(8)]
    ctx = prefix + 256
    rt = base.runtime(max_seqs=n + 2, max_context=ctx, max_rows=512, adapter_slots=8, lora_rank=16,
                      num_pages=prefix // 16 + n * 24 + 32, chunk_pages=chunk_pages)
    pool = KvCachePool(cfg, 64 << 30, "icarus")
    prompt = [int(t) for t in np.random.default_rng(0).integers(1, cfg.vocab_size, prefix)]
    ss = [E.new_session(base, ads[i % 8], ctx, runtime=rt) for i in range(n)]
    toks = [E.prefill(ss[0], prompt, pool=pool)]
    pool.commit(None, prompt, ss[0].cache, next_token_fn=lambda p: E.base_next_token_at(ss[0], p))
    toks += [E.prefill(s, prompt, pool=pool) for s in ss[1:]]
    for _ in range(3):
        toks = E.decode_step_batch(ss, toks)
    torch.cuda.synchronize()
    kind_ms = (C.c_float * 10)()
    _lib.check(rt._lib.icr_profile_step(rt._handle, kind_ms, _lib.stream_handle()))
    names = ("embed", "qkv", "attention", "o", "gate_up", "down", "lm_gather", "lm_head", "argmax")
    print({nm: round(kind_ms[i], 3) for i, nm in enumerate(names)}, "serial total", round(kind_ms[9], 3))
    avg = C.c_float()
    _lib.check(rt._lib.icr_profile_ablate(rt._handle, 0, 10, C.byref(avg), _lib.stream_handle()))
    full = avg.value
    out = {"full_step_ms": round(full, 3)}
    for nm, k in (("qkv", 1), ("attn", 2), ("o", 3), ("gu", 4), ("down", 5), ("lm", 7)):
        _lib.check(rt._lib.icr_profile_ablate(rt._handle, 1 << k, 10, C.byref(avg), _lib.stream_handle()))
        out[nm] = round(full - avg.value, 3)
    print("in-graph marginal ms:", out)
    trace = [a for a in sys.argv[1:] if not a.startswith("--")]
    if trace:
        _lib.check(rt._lib.icr_profile_trace(rt._handle, trace[0].encode(), _lib.stream_handle()))


if __name__ == "__main__":
    cp = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--chunk-pages=")]
    main(chunk_pages=cp[0] if cp else None)
