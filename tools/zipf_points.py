"""Config-5 (Zipf(1.2) over 64 experts, int4) timing at a few token counts through bench.run_point.
usage: python tools/zipf_points.py [T ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_02410_b200 as m  # noqa: E402

Ts = [int(x) for x in sys.argv[1:]] or [64, 512]
for T in Ts:
    r, lay = bench.run_point(m, torch, 64, 1024, 4096, 4, T, 1, 40, 5, torch.device("cuda:0"), 6545.9, 1632.0,
                             n_layers=4 if T >= 4096 else bench.N_LAYERS, zipf=True)
    del lay
    torch.cuda.empty_cache()
    print(json.dumps({"T": T, "ms_per_step": round(r["ms_per_step"], 5), "share": r.get("kernel_share")}))
