import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2111_14641_b200 import _device as D
n, k, nnz, row0, cols, path = [int(x) for x in sys.argv[1:7]]
g = np.random.Generator(np.random.Philox(77))
X = D.to_cm(torch.from_numpy(np.asfortranarray(g.standard_normal((n, cols)))), torch.float64, 'cuda')
a = torch.zeros(k, cols, dtype=torch.float64, device='cuda').t().contiguous().t()
if path == 0:
    D.sketch_sparse_sign(X, row0, 11, k, nnz, a)
else:
    tab = D.sparse_sign_table(11, k, nnz, row0, n, X.device)
    torch.cuda.synchronize()
    print("table ok", flush=True)
    D.sketch_sparse_sign(X, row0, 11, k, nnz, a, table=tab)
torch.cuda.synchronize()
print("ok", n, k, nnz, row0, cols, path)
