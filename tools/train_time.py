"""Device time of bench.py's config-5 training step (FPVS_* A/B switches via env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.train_config5(1, 0, steps=int(os.environ.get("STEPS", "20")))
print(f"{os.environ.get('TAG', '')} config5 step {r['ms_per_step'] * 1e3:.1f} us, loss {r.get('loss_mean')}")
