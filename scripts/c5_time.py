"""bench.py's c5 auxiliary measurement alone (30 sweeps + 10 IPM iterations, one GPU).

python scripts/c5_time.py
"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

if __name__ == "__main__":
    print(json.dumps(bench.aux_c5(torch.device("cuda", 0), 1, 0)), flush=True)
