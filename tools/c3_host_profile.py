"""Host vs device time of the C3 workflow: the wall time of workflow.serve, the summed
icr_forward host split (prep / upload+launch / wait) and a cProfile of the Python side.

  python tools/c3_host_profile.py
"""
import cProfile
import ctypes as C
import io
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import bench
    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import workflow as W
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig
    cfg = ModelConfig(**bench.C2)
    wcfg = W.WorkflowConfig(requests=64, prefix_len=8192, max_batch=64)
    prefix, reqs = W.make_workload(wcfg, cfg.vocab_size)
    need = W.max_context_tokens(prefix, reqs)
    max_ctx = (need + 64 + 15) // 16 * 16
    base = BaseWeights.on_device(cfg, seed=0)
    ads = [AdapterSet.on_device(cfg, 16, 32.0, seed=1 + i, task=f"agent{i}") for i in range(8)]
    lib = _lib.load()
    private_pages = (need - 8192) // 16 + 8
    num_pages = 8192 // 16 + 64 * private_pages + 64
    for it in range(2):
        rt = base.runtime(max_seqs=68, max_context=max_ctx, max_rows=512, adapter_slots=8,
                          lora_rank=16, num_pages=num_pages)
        pool = KvCachePool(cfg, budget_bytes=num_pages * cfg.num_layers * 2 * cfg.kv_dim * 2 * 16,
                           mode="icarus")
        W.warm_prefix(base, pool, prefix, max_ctx, runtime=rt)
        buf = (C.c_double * 4)()
        lib.icr_host_timing(buf, 1)
        pr = cProfile.Profile() if it == 1 else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if pr:
            pr.enable()
        rep = W.serve(base, ads, pool, prefix, reqs, wcfg, max_ctx, runtime=rt)
        if pr:
            pr.disable()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        lib.icr_host_timing(buf, 1)
        n = buf[0]
        print(f"iter {it}: wall {wall:.3f} s ({rep.decode_tok_s:.0f} tok/s), icr_forward calls {n:.0f}: "
              f"prep {buf[1] / 1e6:.3f} s, upload+launch {buf[2] / 1e6:.3f} s, wait {buf[3] / 1e6:.3f} s, "
              f"outside icr_forward {wall - (buf[1] + buf[2] + buf[3]) / 1e6:.3f} s")
        if pr:
            s = io.StringIO()
            pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
            print(s.getvalue()[:5000])
        del rt, pool
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
