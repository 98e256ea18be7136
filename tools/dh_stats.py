import sys, numpy as np, torch
sys.path.insert(0,'.')
import workloads, paper_1105_3829_b200 as mtb
for name, px in (("cfg3", workloads.cfg3_uniform_u16()), ("cfg4", workloads.cfg4_three_gauss_u16())):
    src = torch.from_numpy(px).cuda()
    for r in (7, 15, 31):
        med = mtb.rank_filter(src, r).cpu().numpy()
        H = (med >> 8).astype(np.int32)
        h, w = H.shape
        for th in (1, 16, 64):
            t = H[: (h // th) * th, : (w // 256) * 256].reshape(h // th, th, w // 256, 256).transpose(0, 2, 1, 3).reshape(-1, th * 256)
            d = np.array([len(np.unique(row)) for row in t[:: max(1, len(t) // 2000)]])
            print(name, "r", r, "tile 256x%d" % th, "distinct H mean %.2f max %d" % (d.mean(), d.max()),
                  "| hb spread img", len(np.unique(px[::7, ::7] >> 8)), flush=True)
        # fraction of horizontally adjacent pairs with same H
        print(name, "r", r, "adjacent same H: %.3f" % (H[:, 1:] == H[:, :-1]).mean(), "vertical same: %.3f" % (H[1:] == H[:-1]).mean())
