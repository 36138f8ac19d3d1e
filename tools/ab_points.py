"""Times single decode shapes (bench._decode_point) for quick same-box A/Bs of env settings.
    KVLC_X=... python tools/ab_points.py B:HKV:HQ:N ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda:0")
out = []
for spec in sys.argv[1:]:
    b, hkv, hq, n = (int(x) for x in spec.split(":"))
    out.append(f"{spec} {bench._decode_point(dev, b, hkv, hq, n, 7000.0)['us_per_step']:.2f}")
print(" | ".join(out))
