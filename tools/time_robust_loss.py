"""Time gs_loss_l1_masked with and without the 10x-median rule at 1200x680 (CUDA events)."""
import numpy as np
import torch

import gs_inputs as gi
import paper_2311_11700_b200 as g

W, H = 1200, 680
c, d = gi.random_images(W, H, 1)
tc, td = gi.random_images(W, H, 2)
a = np.ones((H, W), np.float32)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
C, D, TC, TD, A = map(dev, (c, d, tc, td, a))
pipe = g.RenderPipeline(16, 4096, W, H)
dc = torch.zeros(3, H, W, device="cuda")
dd = torch.zeros(H, W, device="cuda")
loss = torch.zeros(1, dtype=torch.float64, device="cuda")
for k in (0.0, 10.0):
    for _ in range(5):
        g.gs_loss_l1_masked(C, D, TC, TD, A, 0.5, k, W, H, 0.9, 0.1, dc, dd, loss, pipe.ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.gs_loss_l1_masked(C, D, TC, TD, A, 0.5, k, W, H, 0.9, 0.1, dc, dd, loss, pipe.ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"outlier_k={k}: {e0.elapsed_time(e1) / 200 * 1000:.1f} us per call")
