import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import gg_inputs as gi, paper_2510_15352_b200 as gg
sc = gi.config_scene('c3'); E, W, H = 4096, 640, 480
cams = gi.cameras(5, E, W, H, sc)
r = gg.Renderer(0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
sid = r.load_scene(t(sc.means), t(sc.scales), t(sc.quats), t(sc.opacities), t(sc.sh), sc.sh_degree)
ids, vm, K = t(np.full(E, sid, np.int32)), t(cams.viewmats), t(cams.intrinsics)
d_rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device='cuda'); d_dep = torch.empty((E, H, W), device='cuda')
opts = gg.default_opts(flags=gg.GG_TIGHT_TILES)
s = torch.cuda.current_stream()
def dev_render():
    gg.gg_render(r.ctx, E, ids, vm, K, W, H, opts, d_rgb, d_dep, None, s)
hr = torch.empty((E, H, W, 3), dtype=torch.uint8).pin_memory(); hd = torch.empty((E, H, W)).pin_memory()
hid, hvm, hK = np.full(E, sid, np.int32), cams.viewmats, cams.intrinsics
hidp, hvmp, hKp = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (hid, hvm, hK)]
def host(pinned):
    a = (hidp, hvmp, hKp) if pinned else (hid, hvm, hK)
    gg.gg_render_host(r.ctx, E, a[0], a[1], a[2], W, H, opts, hr, hd, None, s)
for f, name in ((dev_render, 'device'), (lambda: host(False), 'host (pageable inputs)'), (lambda: host(True), 'host (pinned inputs)')):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.time(); f(); torch.cuda.synchronize(); ts.append(time.time() - t0)
    print(f"{name}: {min(ts)*1e3:.1f} ms", flush=True)
gg.gg_set_timing(r.ctx, True); host(True); torch.cuda.synchronize(); print('stages (host path)', gg.gg_get_stage_ms(r.ctx))
