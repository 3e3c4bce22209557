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
x = torch.empty(8800 * 1024 * 1024 // 4, dtype=torch.float32, device='cuda')
h = torch.empty(x.shape, dtype=torch.float32).pin_memory()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def render():
    gg.gg_render(r.ctx, E, ids, vm, K, W, H, None, d_rgb, d_dep, None, stream=sa)
render(); torch.cuda.synchronize()
t0 = time.time(); render(); torch.cuda.synchronize(); tr = time.time() - t0
t0 = time.time(); h.copy_(x, non_blocking=True); torch.cuda.synchronize(); tc = time.time() - t0
t0 = time.time()
with torch.cuda.stream(sb):
    h.copy_(x, non_blocking=True)
render()
torch.cuda.synchronize(); tb = time.time() - t0
print(f"render {tr*1e3:.0f} ms, copy {tc*1e3:.0f} ms, both {tb*1e3:.0f} ms", flush=True)
# host path: pinned host outputs, host inputs
hr = torch.empty((E, H, W, 3), dtype=torch.uint8).pin_memory(); hd = torch.empty((E, H, W)).pin_memory()
hid, hvm, hK = ids.cpu().pin_memory(), vm.cpu().pin_memory(), K.cpu().pin_memory()
def host():
    gg.gg_render_host(r.ctx, E, hid, hvm, hK, W, H, None, hr, hd, None, stream=sa)
host(); torch.cuda.synchronize()
for ch in (1024, 512, 256):
    gg.gg_reserve(r.ctx, E, W, H, ch); host(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.time(); host(); torch.cuda.synchronize(); ts.append(time.time() - t0)
    print(f"host path chunk={ch}: {min(ts)*1e3:.0f} ms (device render {tr*1e3:.0f} ms)", flush=True)
assert torch.equal(hr, d_rgb.cpu()) and torch.equal(hd, d_dep.cpu())
print("host outputs identical to device outputs", flush=True)
