"""The library's instrumentation (-m gpu): the per-kernel CUDA-event log (gs_ws_set_event_log,
gs_events_*) names every logged launch of one fused config-0 iteration in stream order with a
positive time, and the launch counter (gs_ws_launch_count, bench.py's gpu_launches) counts the 8
kernels of the iteration (the zeroing kernel is counted but not logged)."""
import numpy as np
import pytest
import torch

import gs_inputs as gi
from gpu_helpers import key_cap_for, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_event_log_and_launch_count():
    import paper_2311_11700_b200 as g
    cfg = gi.CONFIGS[0]
    p, v = cfg.scene(), cfg.view()
    n = p.shape[1]
    key_cap, _ = key_cap_for(p, v, cfg.cam)
    pipe = g.RenderPipeline(n, key_cap, cfg.cam.width, cfg.cam.height)
    P, V = to_dev(p), to_dev(v)
    tc, td = (to_dev(x) for x in gi.random_images(cfg.cam.width, cfg.cam.height, 5))
    grad = torch.zeros_like(P)
    gp = torch.zeros(6, dtype=torch.float64, device="cuda")

    def it():
        pipe.iteration(P, n, V, cfg.cam, tc, td, grad, gp, bin_flags=g.GS_FLAG_NO_HOST_SYNC, fwd_flags=0,
                       assign_grads=True, fused_loss=True)
    it()
    torch.cuda.synchronize()
    l0 = pipe.ws.launches()
    log = g.EventLog(pipe.ws, 64)
    with log:
        it()
    torch.cuda.synchronize()
    assert pipe.ws.launches() - l0 == 8
    rows = log.read()
    log.close()
    names = [k for k, _ in rows]
    assert names == ["project", "bin_coop", "bucket_emit", "render_fwd", "sgrad_clear", "render_bwd_tiles",
                     "gaussian_bwd"], names
    assert all(ms > 0 for _, ms in rows) and np.isfinite([ms for _, ms in rows]).all()
