"""Per-GEMM cost breakdown on the C2 decode batch: full fused epilogue vs no LoRA vs a
plain fp32 store (icr_profile_gemm variant bits)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_13281_b200 import _lib  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402


def setup():
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig
    import bench
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
    setup.keep = (base, ads, ss, pool)
    return rt


def main():
    rt = setup()
    avg = C.c_float()
    for which, name in ((0, "o"), (1, "gate_up"), (2, "down"), (3, "lm_head")):
        out = []
        for var, vname in ((0, "full"), (64, "no_shrink"), (16, "no_lora"), (48, "plain")):
            _lib.check(rt._lib.icr_profile_gemm(rt._handle, which | var, 3, C.byref(avg),
                                                _lib.stream_handle()))
            out.append(f"{vname}={avg.value*1e3:7.1f}us")
        print(name, " ".join(out), flush=True)


if __name__ == "__main__":
    main()
