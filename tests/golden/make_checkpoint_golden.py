"""Checkpoint containers written by the UNMODIFIED reference `icarus.checkpoint` (toy shapes of
its own tests/test_checkpoint.py), committed as fixtures for tests/test_checkpoint.py.

Only runnable where /root/reference exists (the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_checkpoint_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")


def main() -> None:
    sys.path.insert(0, str(REF))
    from icarus.checkpoint import save_adapters, save_base
    from icarus.model import AdapterSet, ModelConfig, init_base

    cfg = ModelConfig(num_layers=2, hidden_dim=8, num_heads=2, num_kv_heads=1, head_dim=4,
                      ffn_dim=16, vocab_size=32)
    base = init_base(cfg, seed=1)
    save_base(HERE / "ckpt_base_toy.ckpt", base)
    base64 = init_base(ModelConfig(**{**json.loads(cfg.canonical_json()), "precision": "f64"}), seed=5)
    save_base(HERE / "ckpt_base_toy_f64.ckpt", base64)
    adapters = AdapterSet.init(cfg, rank=3, alpha=6.0, seed=9, task="copy")
    rng = np.random.default_rng(0)
    for per in adapters.layers:
        for pair in per.values():
            pair.b.data = rng.standard_normal(pair.b.shape).astype(cfg.dtype)
    save_adapters(HERE / "ckpt_adapters_toy.ckpt", adapters)
    out = {
        "base_freeze_hash": base.freeze_hash,
        "base_f64_freeze_hash": base64.freeze_hash,
        "sha256": {name: hashlib.sha256((HERE / name).read_bytes()).hexdigest()
                   for name in ("ckpt_base_toy.ckpt", "ckpt_base_toy_f64.ckpt", "ckpt_adapters_toy.ckpt")},
        "adapter_b_sums": [float(pair.b.data.astype(np.float64).sum())
                           for per in adapters.layers for _, pair in sorted(per.items())],
    }
    (HERE / "ckpt_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(json.dumps(out["sha256"], indent=1))


if __name__ == "__main__":
    main()
