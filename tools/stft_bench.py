"""Time the device STFT / iSTFT at the configs' front-end sizes against the
numpy restatement of the reference (oracle/stft_oracle.py) on the host."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import stft_oracle as SO  # noqa: E402
from paper_1903_03237_b200 import istft, stft  # noqa: E402

for name, (n, M, L, hop) in {"c1 (T=1024, M=8, n_fft 1024)": (1023 * 256, 8, 1024, 256),
                             "c3 (T=8192, M=16, n_fft 2048)": (8191 * 256, 16, 2048, 256)}.items():
    x = np.random.default_rng(0).standard_normal((n, M)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    for _ in range(3):
        spec = stft(xd, L, hop)
        y = istft(spec, L, hop, length=n)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 20
    e[0].record()
    for _ in range(reps):
        spec = stft(xd, L, hop)
    e[1].record()
    for _ in range(reps):
        y = istft(spec, L, hop, length=n)
    e[2].record()
    torch.cuda.synchronize()
    ts, ti = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
    t0 = time.perf_counter()
    s_ref = SO.stft(x.astype(np.float64), L, hop)
    t1 = time.perf_counter()
    SO.istft(s_ref, L, hop, length=n)
    t2 = time.perf_counter()
    err = np.linalg.norm(spec.cpu().numpy() - s_ref) / np.linalg.norm(s_ref)
    print(f"{name}: F,T = {spec.shape[0]},{spec.shape[1]}; device stft {ts:.3f} ms, istft {ti:.3f} ms "
          f"(fp32); host numpy stft {1e3 * (t1 - t0):.1f} ms, istft {1e3 * (t2 - t1):.1f} ms (fp64, "
          f"{os.cpu_count()} cores); rel err {err:.1e}", flush=True)
