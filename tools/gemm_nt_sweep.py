"""F32-epilogue GEMM time against the token-tile width (16..256 rows) at the decode shapes,
with and without the tcgen05 MMAs (skip_mma isolates the streaming + tail cost)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = sys.argv[:1]
import tools.gemm_bw as G  # noqa: E402

for M, K in ((4096, 4096), (28672, 4096), (4096, 14336)):
    for rows in (16, 64, 128, 256):
        for skip in (0, 1):
            G.run(M, K, rows, skip=skip)
