"""The four standalone interleave / deinterleave calls of bench.interleave_side at
the config-2 size, once each (for ncu: `ncu --set full -k regex:"il_|deil_"`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    print(bench.interleave_side(reps=int(os.environ.get("REPS", "3"))))
