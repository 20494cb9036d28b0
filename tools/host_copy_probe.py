"""Host-side costs of the numpy decode path (GPU box host)."""
import time

import numpy as np
import torch

B = 1 << 24
a = np.random.default_rng(0).random((B, 2), dtype=np.float32)
px = torch.empty((B, 2)).pin_memory()
po = torch.empty((B, 3)).pin_memory()


def t(name, fn, n=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:50s} {(time.perf_counter() - t0) / n * 1e3:7.2f} ms", flush=True)


t("copy numpy -> pinned (128 MiB)", lambda: px.copy_(torch.from_numpy(a)))
t("aminmax over pinned (128 MiB)", lambda: torch.aminmax(px))
t("np.min / np.max (128 MiB)", lambda: (a.min(), a.max()))
t("np.empty + torch copy pinned -> new (192 MiB)", lambda: torch.from_numpy(np.empty((B, 3), np.float32)).copy_(po))
res = np.empty((B, 3), np.float32)
t("torch copy pinned -> existing (192 MiB)", lambda: torch.from_numpy(res).copy_(po))
t("np.empty + np.copyto (192 MiB)", lambda: np.copyto(np.empty((B, 3), np.float32), po.numpy()))
print("threads", torch.get_num_threads())
