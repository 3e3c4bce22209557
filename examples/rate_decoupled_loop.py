"""Rate-decoupled render loop.

GaussGym steps physics at a control rate and renders at a lower camera rate:
"rendering at the camera rate, not the control rate", 4,096
envs at 50 Hz control / 10 Hz camera.  This loop does the same
with this package:

* the sync-free render (GG_ASYNC) is captured once in a CUDA graph whose
  inputs are fixed device buffers (scene ids, view matrices, intrinsics);
* every `decimation`-th control step copies the current camera poses into
  the graph's input buffer and replays the graph; the other steps reuse the
  held frames;
* each rendered frame batch is converted to the DinoV2 input (gg_dino_input,
  reading R36) for the policy.

Physics is a stand-in (cameras drift along +z of their own frame); the
render path is the product's.  Run: python examples/rate_decoupled_loop.py
[--envs 1024 --steps 50 --decimation 5].
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import gg_inputs as gi  # noqa: E402
import paper_2510_15352_b200 as gg  # noqa: E402


def advance(viewmats: torch.Tensor, dt: float, speed: float = 0.5) -> torch.Tensor:
    """Stand-in physics: move every camera `speed * dt` along its own +z."""
    v = viewmats.clone()
    v[:, 2, 3] -= speed * dt          # world->camera translation of a forward step
    return v


class RateDecoupledRenderer:
    """Graph-captured render of E envs at W x H, replayed on demand."""

    def __init__(self, ctx, scene_ids: torch.Tensor, viewmats: torch.Tensor, intrinsics: torch.Tensor, W: int,
                 H: int, dino_size: int = 224):
        E = scene_ids.numel()
        self.ctx, self.E, self.W, self.H = ctx, E, W, H
        dev = scene_ids.device
        self.ids = scene_ids
        self.vm = viewmats.clone()                   # the graph's fixed input buffer
        self.K = intrinsics
        self.rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device=dev)
        self.depth = torch.empty((E, H, W), dtype=torch.float32, device=dev)
        self.dino = torch.empty((E, 3, dino_size, dino_size), dtype=torch.bfloat16, device=dev)
        # capacities from a synchronous render of the first poses (1.5x the densest chunk seen)
        gg.gg_render(ctx, E, scene_ids, viewmats, intrinsics, W, H, gg.default_opts(flags=gg.GG_TIGHT_TILES))
        gg.gg_reserve_async(ctx, E, W, H, 0, -1.5, 0.0)
        opts = gg.default_opts(flags=gg.GG_ASYNC | gg.GG_TIGHT_TILES)
        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())

        def render():
            gg.gg_render(ctx, E, self.ids, self.vm, self.K, W, H, opts, self.rgb, self.depth, None, self.stream)
            gg.gg_dino_input(ctx, E, W, H, self.rgb, dino_size, self.dino, self.stream)

        with torch.cuda.stream(self.stream):         # warm-up outside the capture
            render()
        torch.cuda.current_stream().wait_stream(self.stream)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            render()

    def render(self, viewmats: torch.Tensor):
        self.vm.copy_(viewmats)
        self.graph.replay()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--envs", type=int, default=1024)
    p.add_argument("--steps", type=int, default=50, help="control steps")
    p.add_argument("--decimation", type=int, default=5, help="control steps per camera frame (50 Hz / 10 Hz)")
    p.add_argument("--gaussians", type=int, default=1_000_000)
    args = p.parse_args()
    E, W, H = args.envs, 640, 480
    sc = gi.room_scene(0, args.gaussians, 3)
    r = gg.Renderer(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    sid = r.load_scene(t(sc.means), t(sc.scales), t(sc.quats), t(sc.opacities), t(sc.sh), sc.sh_degree)
    cams = gi.cameras(1, E, W, H, sc)
    vm = t(cams.viewmats)
    rr = RateDecoupledRenderer(r.ctx, t(np.full(E, sid, np.int32)), vm, t(cams.intrinsics), W, H)
    dt = 1.0 / 50.0
    frames = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        vm = advance(vm, dt)
        if k % args.decimation == 0:
            rr.render(vm)                 # new camera frame; rr.dino holds it until the next one
            frames += E
        # ... policy(rr.dino, proprio) would run here every control step ...
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    gg.gg_check_errors(r.ctx)
    print(f"{args.steps} control steps, {frames} env-frames rendered in {el * 1e3:.1f} ms "
          f"({frames / el:.0f} env-frames/s, {E * args.steps / el:.0f} env-steps/s)")
    r.close()


if __name__ == "__main__":
    main()
