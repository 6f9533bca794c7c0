import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import engine, _native as nat
rng = np.random.default_rng(20240117)
n, h, w = 5, 70, 90
a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
pair = engine.device_pair(ta, tb, 8, True)
res = []
for want in (nat.WANT_CS, nat.WANT_Q | nat.WANT_L | nat.WANT_CS):
    for rep in range(5):
        s, _ = engine.ssim(pair, cfg.window, cfg.c1, cfg.c2, want)
        res.append((want, s.cpu().numpy()[:, 2].copy()))
base = res[0][1]
for want, r in res:
    print(want, np.abs(r - base).max())
# per-frame single calls
for i in range(n):
    p1 = engine.device_pair(ta[i:i+1], tb[i:i+1], 8, True)
    s, _ = engine.ssim(p1, cfg.window, cfg.c1, cfg.c2, nat.WANT_CS)
    print('single', i, s.cpu().numpy()[0, 2] - base[i])
