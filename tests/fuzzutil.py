"""Trial counts of the seeded fuzz loops (GS_FUZZ_SCALE multiplies them for
soak runs on the GPU box; the default is the suite's own count)."""
import os


def fuzz_trials(n: int) -> int:
    return n * max(1, int(os.environ.get("GS_FUZZ_SCALE", "1")))
