import math, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import sfgen, oracle
from sfgen import scene
import paper_2406_18031_b200 as sf
seq = sfgen.config_sequence(1, frames=3, H=96, W=80)
Hc, Wc = 70, 90
f = Wc / (2 * math.tan(math.radians(70.0) / 2)); K = (f, f, (Wc - 1) / 2, (Hc - 1) / 2)
a = math.radians(2.0)
R = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]], np.float32)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
ma = sf.StructureFlow(seq.geom, seq.params, kernel=sf.SF_KERNEL_FUSED)
mb = sf.StructureFlow(seq.geom, seq.params, kernel=sf.SF_KERNEL_FUSED)
for k in range(2):
    Yc, Zc = scene.render_camera(seq.scene, Hc, Wc, K, float(k))
    Ycd, Zcd = dev(Yc[None]), dev(Zc[None])
    sf.sf_step_camera(ma.ctx, Ycd.data_ptr(), Zcd.data_ptr(), Hc, Wc, K, R.flatten())
    Y, D = mb.map_inputs(Ycd, Zcd, K, R)
    mb.step(Y, D)
    torch.cuda.synchronize()
    wa, ra, ya = ma.get_fields(); wb, rb, yb = mb.get_fields(); torch.cuda.synchronize()
    wa, wb, ya, yb, ra, rb = [t[0].cpu().numpy() for t in (wa, wb, ya, yb, ra, rb)]
    for name, a, b in (("w", wa, wb), ("rho", ra, rb), ("yhat", ya, yb)):
        d = np.abs(a.astype(np.float64) - b)
        bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
        print(k, name, "mismatches", int(bad.sum()), "max", np.nanmax(d) if bad.any() else 0, "at", np.argwhere(bad)[:5].tolist() if bad.any() else "")
