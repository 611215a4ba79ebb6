"""Run bench.config4_line alone (prints the JSON)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

if __name__ == "__main__":
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    print(json.dumps(bench.config4_line(flush), indent=1))
