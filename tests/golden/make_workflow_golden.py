"""Golden counters of the reference serving loop (`simulate.run`, src/simulate.py:254-364) on a
C1-sized model, produced by running the UNMODIFIED reference `icarus` package.

Only runnable where /root/reference exists (the build container); the output is committed
next to this script:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_workflow_golden.py

Produces workflow_c1.json: the workload trace (`generate_workload`, src/simulate.py:114-160:
per request the turns' agent, new tokens and output length), and for both pool modes the
RunReport counters plus the pool's final `stats()`. The serving counters depend only on the
trace's lengths and the pool's rules -- not on which tokens the model emits -- so the B200
driver (paper_2603_13281_b200.workflow.serve, continuous batching) must reproduce them
exactly: tests/test_gpu_workflow.py.
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from icarus.model import ModelConfig, init_base  # noqa: E402
from icarus.simulate import CostModel, WorkloadConfig, generate_workload, make_agents, run  # noqa: E402

C1 = dict(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128, ffn_dim=1024,
          vocab_size=1024)


def main() -> None:
    cfg = ModelConfig(**C1)
    base = init_base(cfg, seed=0)
    agents = make_agents(cfg, 4, seed=1)
    wl = WorkloadConfig(num_agents=4, requests=6, qps=2.0, input_len_min=20, input_len_max=40,
                        output_len_min=4, output_len_max=9, obs_len_min=6, obs_len_max=14,
                        turns_min=2, turns_max=4, seed=3)
    trace = generate_workload(wl, vocab_size=cfg.vocab_size, max_context=256)
    budget = 1 << 24
    out = {"model": C1, "workload": dataclasses.asdict(wl), "budget_bytes": budget,
           "trace": [[[t.agent, list(t.new_tokens), t.output_len] for t in r.turns]
                     for r in trace.requests],
           "reports": {}}
    for mode in ("icarus", "baseline"):
        from icarus.kvpool import KvCachePool  # noqa: F401  (the pool run() builds)
        rep = run(trace, mode, base, agents, budget, CostModel(), max_context=256)
        d = dataclasses.asdict(rep)
        for k in ("latencies_ms", "p95_latency_ms", "throughput_rps", "sim_seconds", "qps"):
            d.pop(k)
        out["reports"][mode] = d
    (HERE / "workflow_c1.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out["reports"], indent=1))


if __name__ == "__main__":
    main()
