"""How many (tile, Gaussian) keys the alpha >= 1/255 AABB (the record's ex, ey) would give
versus the 3DGS square rect (R10), garden camera 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, gen
import paper_2510_14564_b200 as bgs
s = gen.garden()
cam = s.cameras[0]
theta = torch.from_numpy(s.theta).cuda()
r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 26)
r.forward(theta, cam, s.sh_degree)
v = r.views()
class P:
    def __init__(s_, p, n, t):
        s_.__cuda_array_interface__ = {"shape": (n,), "typestr": t, "data": (int(p), False), "version": 2}
rec = torch.as_tensor(P(v.record, 12 * s.n, "<f4"), device="cuda").view(s.n, 12)
tt = torch.as_tensor(P(v.tiles_touched, s.n, "<i4"), device="cuda").to(torch.int64)
vis = tt > 0
x, y, ex, ey = rec[:, 0], rec[:, 1], rec[:, 2], rec[:, 3]
TX, TY = (cam.width + 15) // 16, (cam.height + 15) // 16
x0 = torch.clamp(torch.floor((x - ex) / 16), 0, TX); x1 = torch.clamp(torch.floor((x + ex) / 16) + 1, 0, TX)
y0 = torch.clamp(torch.floor((y - ey) / 16), 0, TY); y1 = torch.clamp(torch.floor((y + ey) / 16) + 1, 0, TY)
tight = ((x1 - x0) * (y1 - y0)).clamp(min=0).to(torch.int64)
tight = torch.where(vis & (ex > 0), tight, torch.zeros_like(tight))
print("K square (R10):", int(tt.sum()), " K tight AABB:", int(tight.sum()), " ratio", float(tight.sum()) / float(tt.sum()))
print("visible", int(vis.sum()), " empty level set (o < 1/255):", int((vis & (ex <= 0)).sum()))
