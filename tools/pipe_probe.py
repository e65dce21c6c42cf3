"""Measure FFMA / FFMA2 / MUFU.RSQ throughput on the current GPU (roofline inputs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_16079_b200.device import fp32_peak_gflops  # noqa: E402

torch.cuda.set_device(0)
res = {name: max(fp32_peak_gflops(8192, m) for _ in range(3))
       for m, name in enumerate(("ffma_gflops", "ffma2_gflops", "mufu_rsq_gops"))}
res["sm_count"] = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps(res))
