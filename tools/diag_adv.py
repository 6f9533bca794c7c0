import sys; sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2101_06354_b200 as P
from oracle import ssim_oracle as O
h, w = 120, 520
yy, xx = np.mgrid[0:h, 0:w]
grad = ((xx * 255) // (w - 1)).astype(np.uint8)
a, b = grad, np.clip(grad.astype(int) + 1, 0, 255).astype(np.uint8)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
got = P.ssim_map(a, b, cfg)
want = O.ssim_maps(a, b, shape="gauss", k=11, sigma=1.5)
for name, g, w_ in zip("l cs q".split(), (got.l_map.values, got.cs_map.values, got.q_map.values), want):
    d = np.abs(g - w_); i = np.unravel_index(d.argmax(), d.shape)
    print(name, d.max(), i, g[i], w_[i])
st = P.local_statistics(a, b, cfg.window)
ws = O.local_stats(a, b, shape="gauss", k=11, sigma=1.5) if hasattr(O, "local_stats") else None
print("mu1", st.mu1[0, :4], "var1", st.var1[0, :4], "cov", st.cov[0, :4])
