"""The C-ABI library loads on a CPU-only box and exports every symbol the header declares."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_header_and_binding_agree():
    from paper_2603_13281_b200 import _lib
    header = (ROOT / "include" / "icarus_b200.h").read_text()
    declared = set(re.findall(r"\b(icr_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_lib.EXPORTED)


def test_library_exports_every_symbol():
    from paper_2603_13281_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("library not built")
    lib = _lib.load()
    for name in _lib.EXPORTED:
        assert hasattr(lib, name), name
    assert lib.icr_abi_version() == 2


def test_status_codes_map_to_reference_exceptions():
    from paper_2603_13281_b200 import _lib, errors
    assert _lib._STATUS[1] is errors.ShapeError
    assert _lib._STATUS[2] is errors.ConfigError
    assert _lib._STATUS[3] is errors.ModeError
    assert _lib._STATUS[4] is errors.StateError
    assert _lib._STATUS[5] is errors.CapacityError
    assert _lib._STATUS[6] is errors.ContractViolationError
    assert _lib._STATUS[8] is IndexError


def test_sources_target_sm100a_only():
    from paper_2603_13281_b200 import build
    assert build.ARCH == ["-gencode", "arch=compute_100a,code=sm_100a"]


def test_auto_chunk_pages_rule():
    """Attention chunk length chosen per runtime from its context capacity (fixed per runtime:
    batch invariance): C1/C2 contexts keep 16-page chunks, 4k gets 32, the 8k-prefix workflow
    (C3) and 16k get 64, the 32k context (C4) 128."""
    from paper_2603_13281_b200.runtime import auto_chunk_pages
    assert auto_chunk_pages(1024) == 16
    assert auto_chunk_pages(2418) == 16      # bench.py C2 capacity
    assert auto_chunk_pages(2560) == 16
    assert auto_chunk_pages(2576) == 32
    assert auto_chunk_pages(4112) == 32
    assert auto_chunk_pages(8448) == 64      # tools/c3_step_profile.py capacity
    assert auto_chunk_pages(8976) == 64      # C3 workflow capacity
    assert auto_chunk_pages(16400) == 64     # 16k context: 17 chunks x 8 KV heads fill the SMs
    assert auto_chunk_pages(17424) == 128
    assert auto_chunk_pages(32800) == 128
    assert auto_chunk_pages(1 << 20) == 128


def test_missing_library_or_device_fails_loudly():
    """No CPU fallback: without the built library the product path raises DeviceError, and a
    runtime refuses to start without a CUDA device (this container has none)."""
    import subprocess
    import sys
    code = ("import os, sys\n"
            "os.environ['ICR_LIB_PATH'] = '/nonexistent/libicarus_b200.so'\n"
            "from paper_2603_13281_b200 import _lib\n"
            "from paper_2603_13281_b200.errors import DeviceError\n"
            "try:\n    _lib.load()\nexcept DeviceError:\n    sys.exit(0)\nsys.exit(1)\n")
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    assert subprocess.run([sys.executable, "-c", code], cwd=root).returncode == 0
    import torch
    if not torch.cuda.is_available():
        from paper_2603_13281_b200.errors import DeviceError
        from paper_2603_13281_b200.model import ModelConfig, init_base
        base = init_base(ModelConfig(num_layers=1, hidden_dim=128, num_heads=2, num_kv_heads=1,
                                     head_dim=64, ffn_dim=256, vocab_size=256), seed=0)
        with pytest.raises(DeviceError):
            base.runtime(max_seqs=2, max_context=64)
