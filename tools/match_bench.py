"""Time mrf_dict_match on the MRF-sized problem (65536 voxels x 3336 atoms x 1000 frames)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth.dictionary as sd  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

L, V = 1000, 65536
g = sd.t1t2_grid()
D = sd.surrogate_dictionary(L, g)
dic = binding.Dictionary(D, g)
x = (torch.randn(L, V, dtype=torch.complex64, device="cuda"))
for _ in range(3):
    dic.match(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
s.record()
for _ in range(reps):
    dic.match(x)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
K = D.shape[0]
fl = 8.0 * V * K * L
print(f"match: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s useful (8 V K L), padded GEMM {2.0 * V * 6912 * 2048 / ms / 1e9:.1f} TFLOP/s")
