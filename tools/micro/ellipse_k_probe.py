"""How many of a view's (tile, Gaussian) keys would an exact ellipse-vs-tile test keep?
(R11' emits every tile the alpha >= 1/255 BOX reaches.)  Counts, on the GPU with torch, the
pairs of the sorted lists whose alpha level-set ellipse reaches a pixel centre of the tile
(the margin of common.cuh's ellipse_hits_block)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


class _P:
    def __init__(self, ptr, count, t):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": t, "data": (int(ptr), False), "version": 2}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "garden"
    s = gen.make(name)
    for view in (0,):
        cam = s.cameras[view]
        theta = torch.from_numpy(s.theta).cuda()
        r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 26)
        r.forward(theta, cam, s.sh_degree)
        v = r.views()
        K = r.num_keys
        nt = v.tiles_x * v.tiles_y
        rec = torch.as_tensor(_P(v.record, 12 * s.n, "<f4"), device="cuda").view(s.n, 12)
        vals = torch.as_tensor(_P(v.values_sorted, K, "<i4"), device="cuda").long()
        rg = torch.as_tensor(_P(v.ranges, 2 * nt, "<i4"), device="cuda").view(nt, 2).long()
        cnt = rg[:, 1] - rg[:, 0]
        tile = torch.repeat_interleave(torch.arange(nt, device="cuda"), cnt)
        keep = 0
        byh = torch.zeros(3, 64, dtype=torch.float64)  # [K, kept] by rect rows
        for a in range(0, K, 1 << 23):
            ids, t = vals[a:a + (1 << 23)], tile[a:a + (1 << 23)]
            R = rec[ids]
            mx, my, A, B, C, thr = R[:, 0], R[:, 1], R[:, 4], R[:, 5], R[:, 6], R[:, 11]
            bx0 = (t % v.tiles_x).float() * 16
            by0 = (t // v.tiles_x).float() * 16
            bx1, by1 = bx0 + 15, by0 + 15
            lx, hx, ly, hy = bx0 - mx, bx1 - mx, by0 - my, by1 - my
            in_x = (lx <= 0) & (hx >= 0)
            in_y = (ly <= 0) & (hy >= 0)
            best = torch.full_like(mx, -3e38)
            dx = torch.where(lx > 0, lx, hx)
            dy = torch.clamp(-B * dx / (2 * C), ly, hy)
            best = torch.where(~in_x, torch.maximum(best, A * dx * dx + B * dx * dy + C * dy * dy), best)
            dy = torch.where(ly > 0, ly, hy)
            dx = torch.clamp(-B * dy / (2 * A), lx, hx)
            best = torch.where(~in_y, torch.maximum(best, A * dx * dx + B * dx * dy + C * dy * dy), best)
            ex, ey = torch.maximum(-lx, hx), torch.maximum(-ly, hy)
            margin = 1e-3 + 1e-5 * (A.abs() * ex * ex + C.abs() * ey * ey)
            hit = (in_x & in_y) | (best >= thr - margin)
            keep += int(hit.sum())
            ey_ = R[:, 3]
            rows = (torch.floor((my + ey_) / 16) - torch.floor((my - ey_) / 16) + 1).clamp(1, 63).long()
            byh[0] += torch.bincount(rows, minlength=64).double().cpu()[:64]
            byh[1] += torch.bincount(rows, weights=hit.double(), minlength=64).cpu()[:64]
        print(f"{name} view {view}: K {K}  ellipse-kept {keep}  ({keep / K:.3f})", flush=True)
        cum = 0.0
        for h in range(1, 64):
            if byh[0, h] == 0:
                continue
            cum += byh[0, h] - byh[1, h]
            if h <= 8 or h % 8 == 0:
                print(f"   rows {h:2d}: keys {byh[0, h] / K:.3f}  dropped {(byh[0, h] - byh[1, h]) / K:.4f}  cum dropped {cum / K:.4f}")


if __name__ == "__main__":
    main()
