"""Dev probe: how often CUDA's double pow (libdevice, what k_place.cu uses
for interference exponents other than 0.5 / 1 / 2) differs from glibc's pow
(what the reference's `excess ** exponent` calls), over random
(excess, exponent) draws in the placement's range."""
import numpy as np
import torch

rng = np.random.default_rng(0)
N = 4_000_000
x = np.concatenate([rng.uniform(1e-9, 2.0, N // 2), rng.uniform(0, 1, N // 2) ** 3])
e = rng.uniform(0.5, 2.0, N)
cpu = np.array([a ** b for a, b in zip(x[:200000].tolist(), e[:200000].tolist())])
gpu = torch.pow(torch.from_numpy(x[:200000]).cuda(), torch.from_numpy(e[:200000]).cuda()).cpu().numpy()
d = (cpu.view(np.int64) - gpu.view(np.int64))
print(f"CUDA pow vs glibc pow: {np.count_nonzero(d)} of {d.size} differ; max |ulp| {np.abs(d).max()}")
