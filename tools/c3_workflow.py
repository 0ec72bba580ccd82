"""C3 (BASELINE.json configs[2]): multi-agent workflow, 8 adapters chaining on a shared 8k
prefix with cross-model prefix-cache reuse, batch 64 -- Llama-3-8B-shape random-init model on
one B200, continuous batching over the fused multi-model step (paper_2603_13281_b200.workflow).

  python tools/c3_workflow.py [--requests 64] [--prefix 8192] [--layers 32] [--out file.json]

Prints one JSON line: decode tok/s over the whole serving run (prefills of every turn
included in the wall time), request P95 latency (nearest rank), prefix-hit / prefill tokens.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--prefix", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--chunk-pages", type=int, default=None, help="default: the runtime's auto rule")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2603_13281_b200 import workflow as W
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig

    shape = dict(bench.C2)
    shape["num_layers"] = args.layers
    cfg = ModelConfig(**shape)
    wcfg = W.WorkflowConfig(requests=args.requests, prefix_len=args.prefix, max_batch=args.requests)
    prefix, reqs = W.make_workload(wcfg, cfg.vocab_size)
    need = W.max_context_tokens(prefix, reqs)
    max_ctx = (need + 64 + 15) // 16 * 16
    base = BaseWeights.on_device(cfg, seed=0)
    adapters = [AdapterSet.on_device(cfg, 16, 32.0, seed=1 + i, task=f"agent{i}") for i in range(8)]
    private_pages = (need - args.prefix) // 16 + 8
    num_pages = args.prefix // 16 + args.requests * private_pages + 64
    rt = base.runtime(max_seqs=args.requests + 4, max_context=max_ctx, max_rows=512, adapter_slots=8,
                      lora_rank=16, num_pages=num_pages, chunk_pages=args.chunk_pages)
    pool = KvCachePool(cfg, budget_bytes=num_pages * cfg.num_layers * 2 * cfg.kv_dim * 2 * 16,
                       mode="icarus")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    W.warm_prefix(base, pool, prefix, max_ctx, runtime=rt)
    torch.cuda.synchronize()
    prefix_s = time.perf_counter() - t0
    rep = W.serve(base, adapters, pool, prefix, reqs, wcfg, max_ctx, runtime=rt)
    line = {
        "workload": f"C3: {args.requests} requests sharing a {args.prefix}-token prefix, 8 rank-16 "
                    f"adapters round-robin over 2-4 turns, {args.layers}-layer Llama-3-8B shape",
        "decode_tok_s": rep.decode_tok_s, "p95_request_latency_ms": rep.p95_latency_ms,
        "wall_s": rep.wall_s, "prefix_prefill_s": prefix_s, "completed": rep.completed,
        "turns": rep.turns, "decode_steps": rep.decode_steps, "decoder_tokens": rep.decoder_tokens,
        "prefill_tokens": rep.prefill_tokens, "prefix_hit_tokens": rep.prefix_hit_tokens,
        "cross_model_hit_tokens": rep.cross_model_hit_tokens, "max_live": rep.max_live,
        "max_context": max_ctx, "chunk_pages": rt.chunk_pages,
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))


if __name__ == "__main__":
    main()
