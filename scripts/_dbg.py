import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2204_06666_b200 as E
from paper_2204_06666_b200 import workloads as W, distributed as D, _lib as L
from oracle import c_oracle
n, r, c, v = W.permute_symmetric(*W.stencil27(40, 40, 40), seed=4)
m = E.CooMatrix(n, n, r, c, v)
e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(600, 32, 4096))
x = W.deterministic_vector(n, 6)
xr = E.permute_vector(x, e.plan)
want = c_oracle.spmv_ehyb(e, xr)
plan = D.plan_for(e, 0, 1)
A = D.DistributedEhyb(e, device=0, plan=plan)
print('info', {k: v for k, v in L.DevInfo.__dict__.items()} if False else '')
x_ext = A.new_ext(); x_ext[:plan.local_rows] = torch.from_numpy(xr)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
def run(names):
    y = torch.zeros(plan.local_rows, dtype=torch.float64, device='cuda:0')
    for nm in names:
        L.call(nm, A._h, C.c_void_p(x_ext.data_ptr()), C.c_void_p(y.data_ptr()), L.MODE_STRICT, st)
    torch.cuda.synchronize()
    return y.cpu().numpy()
vec = e.params.vec_cache_size
er_rows = set(np.asarray(e.plan.y_idx_er).tolist())
for names in (['ehyb_dev_spmv'], ['ehyb_dev_spmv_ell'], ['ehyb_dev_spmv_ell', 'ehyb_dev_spmv_er'], ['ehyb_dev_spmv_ell', 'ehyb_dev_spmv_er']):
    y = run(names)
    bad = np.flatnonzero(y != want)
    print(names, 'bad', bad.size, bad[:10], 'parts', np.unique(bad // vec)[:10], 'er-rows among bad', sum(int(b) in er_rows for b in bad[:200]))
    if bad.size:
        i = bad[0]; print('  y', y[i], 'want', want[i], 'diff', y[i]-want[i])
