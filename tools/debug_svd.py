import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1108_5359_b200 import matcore, engine
rng = np.random.default_rng(2)
for shape in [(20, 10), (10, 20), (20, 20), (80, 60)]:
    m = rng.standard_normal(shape)
    t = torch.from_numpy(m).cuda()
    u, s, v = engine.svd_device(t)
    s_ref = np.linalg.svd(m, compute_uv=False)
    un, sn, vn = u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
    rec = (un * sn) @ vn.T
    print(shape, 'sigma err', np.abs(sn - s_ref).max(), 'rec err', np.abs(rec - m).max(), 'uTu', np.abs(un.T @ un - np.eye(un.shape[1])).max(), 'vTv', np.abs(vn.T@vn - np.eye(vn.shape[1])).max())
    print('  sn', sn[:4], 'ref', s_ref[:4])
