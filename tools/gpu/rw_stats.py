"""Raster work statistics from an instrumented build (-DGG_RW_STATS, libgg_stats.so):
kept (record, warp) iterations, those no live pixel passes (vote failures), those no
pixel passes even ignoring saturation (geometric failures), mean live pixels per kept
record.  python tools/gpu/rw_stats.py [envs=512]   (GG_LIB must point at libgg_stats.so)
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import gg_inputs as gi  # noqa: E402
import paper_2510_15352_b200 as gg  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 512
wl = gi.Workload("c3", n_envs=E, n_sets=1)
W, H = wl.width, wl.height
r = gg.Renderer(0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
sid = {}
for k, sc in wl.scenes():
    sid[k] = r.load_scene(t(sc.means), t(sc.scales), t(sc.quats), t(sc.opacities), t(sc.sh), sc.sh_degree)
ids = t(np.array([sid[int(k)] for k in wl.binding], np.int32))
rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda")
L = gg.load_library()
L.gg_debug_rw_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 8)()
r.render(ids, t(wl.viewmats[0]), t(wl.intrinsics), W, H, rgb=rgb, depth=dep, flags=gg.GG_TIGHT_TILES)
torch.cuda.synchronize()
L.gg_debug_rw_stats(buf, 1)
r.render(ids, t(wl.viewmats[0]), t(wl.intrinsics), W, H, rgb=rgb, depth=dep, flags=gg.GG_TIGHT_TILES)
torch.cuda.synchronize()
L.gg_debug_rw_stats(buf, 0)
kept, vfail, gfail, live = (int(buf[i]) for i in range(4))
print(json.dumps({"envs": E, "kept_record_warp_iterations": kept, "vote_fail_frac": vfail / max(kept, 1),
                  "geometric_fail_frac": gfail / max(kept, 1), "saturation_fail_frac": (vfail - gfail) / max(kept, 1),
                  "mean_live_pixels_per_kept": live / max(kept, 1),
                  "kept_per_env_frame": kept / E}))
r.close()
