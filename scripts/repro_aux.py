"""Run bench.py's auxiliary configs in one process (c2 time-to-tolerance, then c5) with
tracebacks, optionally after a c4 warm step -- reproduces cross-config interactions.

python scripts/repro_aux.py [--c4]
"""
import json
import sys
import traceback

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
for name, fn in (("c2", lambda: bench.aux_c2(dev)), ("c5", lambda: bench.aux_c5(dev, 1, 0))):
    try:
        print(name, json.dumps(fn()), flush=True)
    except Exception:  # noqa: BLE001
        traceback.print_exc()
        sys.exit(1)
