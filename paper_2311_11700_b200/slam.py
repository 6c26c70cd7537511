"""Parallel tracking and mapping ("in the parallel camera tracking phase";
SURVEY.md §8(f) NEXT-4).

Two host threads, each with its own CUDA stream and its own workspaces, share one GPU:

  tracking (caller's thread, stream ts)   per frame: gs_image_half (coarse target) ->
      Frontend.track_frame (constant-velocity init, coarse-to-fine tracking on the observed area
      with the 10x-median rejection, keyframe rule) against the latest published map snapshot
  mapping (worker thread, stream ms)      per keyframe: adaptive expansion from the new keyframe
      (one ShardedMapper step with GS_DENSIFY_ADD: Eq. 8 candidates, append, prune), then
      `map_iters - 1` steps over a window of K keyframes (the new one plus up to K - 1 random
      earlier ones), then publish a snapshot

The map the tracker reads is a snapshot: two [14][cap] buffers, the tracker on one, the mapper
publishing into the other. The hand-over is stream-ordered with CUDA events and never waits on
the host: the mapper's copy waits for the event the tracker recorded when it last left that
buffer; the tracker waits for the event recorded after the copy. A host lock only guards which
buffer is pending. With `parallel=False` the mapping of a keyframe runs to completion, on the
caller's thread, before the next frame is tracked (the same schedule every run).
"""
from __future__ import annotations

import dataclasses
import queue
import random
import threading

import torch

from . import gs_image_half
from .mapping import Keyframe, ShardedMapper, SplitClone
from .tracking import Frontend, FrontendConfig, Tracker


@dataclasses.dataclass
class SlamConfig:
    frontend: FrontendConfig = dataclasses.field(default_factory=FrontendConfig)
    map_iters: int = 30        # mapping iterations per keyframe (PAPER.md:937 uses 100 on Replica)
    window: int = 10           # K keyframes per mapping iteration
    max_add: int | None = None  # Eq. 8 candidates per keyframe (default H W / 2: the first frame fills)
    parallel: bool = True
    seed: int = 0              # window sampling
    degenerate: tuple[float, float] | None = None   # Eq. 9 (eta, gamma) in the expansion step (NEXT-2)
    sh_degree: int = 0         # 1: the paper's degree-1 SH colour (23 parameter rows, NEXT-1)
    ba: bool = True            # keyframe poses refined in the window's second half (Eq. 13)
    split_clone: SplitClone | None = dataclasses.field(default_factory=SplitClone)


class SlamSystem:
    def __init__(self, cam, n_cap: int, key_cap_full: int, key_cap_half: int, cfg: SlamConfig = SlamConfig(),
                 device="cuda"):
        self.cam, self.cfg = cam, cfg
        dev = torch.device(device)
        self.dev = dev
        self.ts = torch.cuda.Stream(dev)
        self.ms = torch.cuda.Stream(dev)
        max_add = cfg.max_add or (cam.width * cam.height) // 2
        rows = 23 if cfg.sh_degree == 1 else 14
        with torch.cuda.stream(self.ms):
            self.mapper = ShardedMapper(torch.zeros(rows, n_cap, device=dev), 0, [], cam, key_cap_full,
                                        max_add_per_kf=max_add, densify=True, degenerate=cfg.degenerate,
                                        split_clone=cfg.split_clone)
        with torch.cuda.stream(self.ts):
            self.tracker = Tracker(n_cap, key_cap_full, key_cap_half, cam, device)
            self.frontend = Frontend(self.tracker, cfg.frontend)
            half = cam.half()
            self.ch = torch.zeros(3, half.height, half.width, device=dev)
            self.dh = torch.zeros(half.height, half.width, device=dev)
        self.snap = [torch.zeros(rows, n_cap, device=dev) for _ in range(2)]
        self.snap_n = [0, 0]
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.released = [torch.cuda.Event(), torch.cuda.Event()]
        self.front = 0              # snapshot the tracker reads
        self.pending = None         # (buffer, n) published and not yet taken
        self.lock = threading.Lock()
        self.keyframes: list[Keyframe] = []
        self.rng = random.Random(cfg.seed)
        self.poses: list[torch.Tensor] = []
        self.kf_flags: list[bool] = []
        self.map_rounds = 0
        self.jobs: queue.Queue = queue.Queue()
        self.error: BaseException | None = None
        self.worker = None
        if cfg.parallel:
            self.worker = threading.Thread(target=self._map_loop, name="gs-mapping", daemon=True)
            self.worker.start()

    # ------------------------------------------------------------------ mapping side (stream ms)
    def _map_keyframe(self, kf: Keyframe, produced: torch.cuda.Event):
        m = self.mapper
        with torch.cuda.stream(self.ms):
            self.ms.wait_event(produced)   # the keyframe's pose and images (tracking stream)
            if not self.keyframes:
                kf.fixed = True    # the first keyframe anchors the world frame (its pose is never moved)
            self.keyframes.append(kf)
            m.it = 0   # per-keyframe learning-rate schedule (PAPER.md:931-933 over the mapping iterations)
            m.densify = True
            m.ba_iters = None
            m.set_keyframes([kf])   # expansion from the new keyframe only (Eq. 8, "at every keyframe")
            m.step()
            m.densify = False
            older = self.keyframes[:-1]
            window = [kf] + self.rng.sample(older, min(self.cfg.window - 1, len(older)))
            m.set_keyframes(window)
            # bundle adjustment over the window (Eq. 13): the map alone in the first
            # half of the iterations, map and keyframe poses in the second; the first-order SH
            # coefficients are optimised only here
            m.ba_iters = self.cfg.map_iters if self.cfg.ba else None
            for _ in range(self.cfg.map_iters - 1):
                m.step()
            m.ba_iters = None
            self._publish()
            self.map_rounds += 1

    def _publish(self):
        with self.lock:
            b = 1 - self.front
            self.pending = None   # a pending snapshot in b is being overwritten: withdraw it
        n = self.mapper.n
        self.ms.wait_event(self.released[b])   # the tracker's last reads of b are done
        self.snap[b][:, :n].copy_(self.mapper.P[:, :n])
        self.ready[b].record(self.ms)
        with self.lock:
            self.snap_n[b] = n
            self.pending = b

    def _map_loop(self):
        # the worker lives until the None sentinel and marks every job done, so join() never blocks;
        # after a failure the remaining jobs are skipped and the error surfaces in process() / finish()
        while True:
            job = self.jobs.get()
            try:
                if job is None:
                    return
                if self.error is None:
                    self._map_keyframe(*job)
            except BaseException as e:
                self.error = e
            finally:
                self.jobs.task_done()

    # ------------------------------------------------------------------ tracking side (stream ts)
    def _take_snapshot(self):
        with self.lock:
            b = self.pending
            self.pending = None
            if b is None:
                return
            self.released[self.front].record(self.ts)   # tracker leaves the old snapshot here
            self.ts.wait_event(self.ready[b])
            self.front = b

    def _submit(self, kf: Keyframe):
        produced = torch.cuda.Event()
        produced.record(self.ts)
        if self.cfg.parallel:
            self.jobs.put((kf, produced))
        else:
            self._map_keyframe(kf, produced)

    def _check(self):
        if self.error is not None:
            raise RuntimeError("mapping thread failed") from self.error

    def process(self, color: torch.Tensor, depth: torch.Tensor, pose: torch.Tensor | None = None):
        """Track one RGB-D frame (device [3][H][W] colour, [H][W] depth) and, on a keyframe, hand it
        to the mapper. The first frame needs its pose (world->camera 3x4) and becomes a keyframe;
        tracking of the second frame waits for its map. Returns (pose, keyframe?)."""
        self._check()
        cam = self.cam
        caller = torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(self.ts):
            self.ts.wait_stream(caller)   # the frame's producer
            if not self.poses:
                V, kf_flag = pose.to(self.dev, torch.float32).clone(), True
                self.frontend.add_pose(V, keyframe=True)
            else:
                self._take_snapshot()
                gs_image_half(color, depth, cam.width, cam.height, self.ch, self.dh)
                P, n = self.snap[self.front], self.snap_n[self.front]
                V, kf_flag, _ = self.frontend.track_frame(P, n, self.ch, self.dh, color, depth)
            self.poses.append(V)
            self.kf_flags.append(kf_flag)
            if kf_flag:
                self._submit(Keyframe(V.clone(), color.clone(), depth.clone()))
            if len(self.poses) == 1 and self.cfg.parallel:   # the first map must exist before tracking
                self.jobs.join()
                self._check()
        caller.wait_stream(self.ts)
        return V, kf_flag

    def finish(self):
        """Drain the mapping queue and stop the worker; the map (mapper.P[:, :mapper.n]) is final."""
        if self.worker is not None:
            self.jobs.join()
            self.jobs.put(None)
            self.worker.join()
            self.worker = None
        self._check()
        torch.cuda.current_stream(self.dev).wait_stream(self.ms)
        torch.cuda.current_stream(self.dev).wait_stream(self.ts)
