"""Per-config call times (BASELINE configs[0..3], bench.time_configs) for the library in use
(NRNG_LIB_OVERRIDE selects an A/B build).  python tools/cfg_ab.py [--sweep-calls N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1004_3105_b200 as P  # noqa: E402

calls = int(sys.argv[sys.argv.index("--sweep-calls") + 1]) if "--sweep-calls" in sys.argv else 200
big = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
pk = bench.load_probe_peaks()
res = bench.time_configs(P, torch, big, pk["hbm_write_gbs_sustained"], pk["fp64_dfma_per_s_sustained"], calls)
lib = os.path.basename(os.environ.get("NRNG_LIB_OVERRIDE", "default"))
print(lib, " ".join("%s=%.1f" % (k.replace("C4_", "").replace("_n", ":"), v["us_per_call"]) for k, v in res.items()))
