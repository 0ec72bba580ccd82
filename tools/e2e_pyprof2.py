"""cProfile of the public-API decode loop (C2 batch, decode_step_batch back to back)."""
import cProfile
import io
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402


def main():
    from paper_2603_13281_b200 import engine as E
    pv.setup()
    _, _, ss, _ = pv.setup.keep
    toks = [1] * len(ss)
    for _ in range(3):
        toks = E.decode_step_batch(ss, toks)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(64):
        toks = E.decode_step_batch(ss, toks)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue()[:6000])


if __name__ == "__main__":
    main()
