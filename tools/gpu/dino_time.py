"""Time gg_dino_input (u8 frames -> bf16 DinoV2 input, R36) on c3-sized frames.

  python tools/gpu/dino_time.py [envs=4096]   -> one JSON line (ms per call, GB/s moved)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2510_15352_b200 as gg  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
W, H, S = 640, 480, 224
r = gg.Renderer(0)
g = torch.Generator(device="cuda").manual_seed(5)
rgb = torch.randint(0, 256, (E, H, W, 3), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty((E, 3, S, S), dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    gg.gg_dino_input(r.ctx, E, W, H, rgb, S, out, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record(s)
for _ in range(n):
    gg.gg_dino_input(r.ctx, E, W, H, rgb, S, out, s)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
moved = E * (H * W * 3 + 3 * S * S * 2)   # whole frame read once (upper bound) + output written
print(json.dumps({"envs": E, "ms_per_call": ms, "frame_plus_out_GB": moved / 1e9,
                  "GBps_upper": moved / 1e9 / (ms / 1e3)}))
r.close()
