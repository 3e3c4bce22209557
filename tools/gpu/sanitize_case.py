"""Small cases that exercise every shared-memory protocol of libgg, for
`compute-sanitizer --tool racecheck|synccheck|memcheck` (one tool per gpurun call):

  * c1 (20k Gaussians, 4 envs, 64x48) with the paper rects, the opacity-aware
    rects (R35) and the ellipse masks (R37): project, the 3 depth passes
    (warp-private stamp ranking), the <= 256-tile placement (TB = 8 stamps),
    raster_warp_kernel's per-warp srec staging, raster_kernel<COUNTERS>;
  * 640x480 (1,200 tiles: TB = 11 stamp path) and 1024x640 (2,560 tiles: the
    TB = 13 ballot multisplit) on a 20k-Gaussian room;
  * a 7,000-record env (more than one 6,144-record sort block);
  * the GG_ASYNC path (LOOP kernels with work counters, device-built tables);
  * depth-only and RGB-only renders.
Prints one line per case; exits non-zero on any GG error.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import gg_inputs as gi  # noqa: E402
import paper_2510_15352_b200 as gg  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    big = gi.room_scene(3, 60_000, 3, L=8.0, stairs=True)
    bid = r.load_scene(dev(big.means), dev(big.scales), dev(big.quats), dev(big.opacities), dev(big.sh),
                       big.sh_degree)

    def render(scene, sid_, E, W, H, flags=0, rgb=True, depth=True, seed=1):
        cams = gi.cameras(seed, E, W, H, scene)
        ids = dev(np.full(E, sid_, np.int32))
        o_rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8, device="cuda") if rgb else None
        o_d = torch.zeros((E, H, W), device="cuda") if depth else None
        gg.gg_render(r.ctx, E, ids, dev(cams.viewmats), dev(cams.intrinsics), W, H, gg.default_opts(flags=flags),
                     o_rgb, o_d, None)
        gg.gg_check_errors(r.ctx)
        torch.cuda.synchronize()
        return cams

    for name, flags in (("paper", 0), ("tight", gg.GG_TIGHT_TILES), ("ellipse", gg.GG_ELLIPSE_TILES),
                        ("counters", gg.GG_COUNTERS)):
        render(sc, sid, 4, 64, 48, flags)
        print("c1", name, "ok", flush=True)
    render(sc, sid, 2, 64, 48, rgb=False)
    print("c1 depth-only ok", flush=True)
    render(sc, sid, 2, 64, 48, depth=False)
    print("c1 rgb-only ok", flush=True)
    render(big, bid, 2, 640, 480, gg.GG_TIGHT_TILES)
    print("640x480 (TB=11) ok", flush=True)
    render(big, bid, 1, 1024, 640, 0)
    print("1024x640 (TB=13) ok", flush=True)
    gg.gg_reserve_async(r.ctx, 8, 64, 48, 0, 0.9, 6.0)
    render(sc, sid, 8, 64, 48, gg.GG_ASYNC | gg.GG_TIGHT_TILES)
    print("c1 async ok", flush=True)
    r.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
