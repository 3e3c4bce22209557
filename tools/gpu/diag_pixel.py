"""Diagnose non-exempt parity failures of a full-size workload (GPU vs oracle).

  python tools/gpu/diag_pixel.py [cfg] [tight]

Renders the workload as tests/test_gpu_fullsize.py does, finds pixels outside
tolerance on the 8 sampled envs, and for each prints the GPU and oracle
values and replays the pixel's list from the oracle's projected records:
f64 compositing (the oracle's O4) next to an f32 emulation of the kernel's
arithmetic, flagging steps whose decision (cutoff / stop) differs.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import gg_inputs as gi  # noqa: E402
import oracle  # noqa: E402
import paper_2510_15352_b200 as gg  # noqa: E402
from parity import pixel_failures  # noqa: E402
from test_gpu_fullsize import samples  # noqa: E402

f32 = np.float32


def replay(o, px, py, W):
    TX = (W + 15) // 16
    t = (py // 16) * TX + px // 16
    a, b = o.ranges[t]
    gids = o.sorted_gid[a:b]
    P = o.proj
    cx, cy = px + 0.5, py + 0.5
    T, T32 = 1.0, f32(1.0)
    stop64 = stop32 = False
    print(f"  tile {t}: {b - a} records")
    for k, g in enumerate(gids):
        u, v, A, B, C, z = (float(P[g, i]) for i in (1, 2, 3, 4, 5, 6))
        op = float(P[g, 15])
        dx, dy = u - cx, v - cy
        q = max(A * dx * dx + 2 * B * dx * dy + C * dy * dy, 0.0)
        al = min(0.99, op * np.exp(-0.5 * q))
        # f32 emulation (log2 domain as the kernel; FMA order approximate)
        kq = f32(-0.72134752044448170)
        x32 = f32(f32(A) * kq) * f32(dx) * f32(dx) + f32(f32(2) * f32(B) * kq) * f32(dx) * f32(dy) + \
            f32(f32(C) * kq) * f32(dy) * f32(dy) + f32(np.log2(op))
        x32 = min(f32(x32), f32(-0.014499569695115089))
        pass32 = x32 >= f32(-7.99435343685885793)
        al32 = f32(2.0) ** x32 if pass32 else f32(0)
        pass64 = al >= 1 / 255
        note = []
        if pass64 != bool(pass32):
            note.append(f"CUTOFF DIFFERS (al64*255={al * 255:.7f}, x32={x32:.7f})")
        if not stop64 and pass64:
            Tn = T * (1 - al)
            if Tn < 1e-4:
                stop64 = True
                note.append(f"stop64 (Tn={Tn:.6e})")
            else:
                T = Tn
        if not stop32 and pass32:
            Tn32 = f32(T32 - f32(al32 * T32))
            if Tn32 < f32(1e-4):
                stop32 = True
                note.append(f"stop32 (Tn32={Tn32:.6e})")
            else:
                T32 = Tn32
        if note or (pass64 and al > 0.3):
            print(f"   #{k:4d} gid {g:8d} z={z:.6f} o={op:.4f} q={q:.4f} al={al:.6f} T64={T:.6e} T32={T32:.6e} "
                  + " ".join(note))
        if stop64 and stop32:
            break


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    tight = len(sys.argv) > 2 and sys.argv[2] == "tight"
    wl = gi.Workload(cfg)
    E, W, H = wl.n_envs, wl.width, wl.height
    r = gg.Renderer(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    sid, kept = {}, {}
    img = samples(E, 8, 1)
    keep = {int(wl.binding[e]) for e in img}
    for k, sc in wl.scenes():
        sid[k] = r.load_scene(t(sc.means), t(sc.scales), t(sc.quats), t(sc.opacities), t(sc.sh), sc.sh_degree)
        if k in keep:
            kept[k] = sc
    ids = t(np.array([sid[int(k)] for k in wl.binding], np.int32))
    rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
    dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda")
    fl = gg.GG_TIGHT_TILES if tight else 0
    r.render(ids, t(wl.viewmats[0]), t(wl.intrinsics), W, H, rgb=rgb, depth=dep, flags=fl)
    torch.cuda.synchronize()
    for e in img:
        k = int(wl.binding[e])
        osc = oracle.OracleScene.from_inputs(kept[k])
        o = oracle.render_env(osc, wl.viewmats[0][e], wl.intrinsics[e], W, H, flags=oracle.F_TIGHT if tight else 0)
        g_rgb, g_dep = rgb[e].cpu().numpy(), dep[e].cpu().numpy()
        bad = pixel_failures(g_rgb, g_dep, None, o) & ~o.exempt
        for py, px in zip(*np.nonzero(bad)):
            print(f"env {e} pixel ({px},{py}): gpu rgb {g_rgb[py, px]} depth {g_dep[py, px]!r}; oracle rgb "
                  f"{o.rgb[py, px] * 255} depth {o.depth[py, px]!r} alpha {o.alpha[py, px]!r} n_eval "
                  f"{o.n_eval[py, px]} n_contrib {o.n_contrib[py, px]}")
            rel = abs(g_dep[py, px] - o.depth[py, px]) / max(o.depth[py, px], 1e-30)
            print(f"  rgb err {np.abs(g_rgb[py, px] / 255 - np.clip(o.rgb[py, px], 0, 1)).max():.6f} depth rel {rel:.3e}")
            replay(o, px, py, W)
    r.close()


if __name__ == "__main__":
    main()
