"""Probe: the config-2 iteration captured in a CUDA graph vs stream launches."""
import sys, time
import torch
sys.path.insert(0, "/root/repo")
import gs_inputs as gi
import paper_2311_11700_b200 as g

cfg = gi.CONFIGS[2]
cam = cfg.cam
p, v = cfg.scene(), cfg.view()
n = p.shape[1]
P = torch.as_tensor(p, device="cuda"); V = torch.as_tensor(v, device="cuda")
pipe = g.RenderPipeline(n, 60_000_000, cam.width, cam.height)
Pt = torch.as_tensor(gi.gaussians(n, 4, cfg.lo, cfg.hi), device="cuda")
fr = pipe.forward(Pt, n, V, cam)
tc, td = fr.color.clone(), fr.depth.clone()
grad = torch.zeros_like(P)
gp = torch.zeros(6, dtype=torch.float64, device="cuda")
flags = g.GS_FLAG_NO_HOST_SYNC
def step():
    pipe.iteration(P, n, V, cam, tc, td, grad, gp, bin_flags=flags, fwd_flags=0, assign_grads=True, fused_loss=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(5):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
def timeit(fn, k=50):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
t_stream = timeit(step)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
torch.cuda.synchronize()
t_graph = timeit(graph.replay)
step(); torch.cuda.synchronize()
a = grad.clone(); la = pipe.loss.clone()
step(); torch.cuda.synchronize()
b = grad.clone()
graph.replay(); torch.cuda.synchronize()
c = grad.clone(); lc = pipe.loss.clone()
def rel(x, y):
    d = (x - y).abs()
    return float(d.max()), float((d / (y.abs() + 1e-6)).max()), float((d > 2e-3 * y.abs() + 1e-6).float().mean())
print(f"stream {t_stream:.4f} ms  graph {t_graph:.4f} ms")
print("stream vs stream", rel(b, a), " graph vs stream", rel(c, a), " loss", la.item(), lc.item())
