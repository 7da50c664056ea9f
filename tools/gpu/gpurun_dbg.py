import sys, numpy as np, torch, traceback
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
from conftest import Golden
from paper_2101_08825_b200 import assemble
g = Golden("quad_q1_lmax3")
mesh, space, kp, cfg = g.build()
A = assemble(mesh, space, kp, cfg)
torch.cuda.synchronize()
print("nnz", A.nnz, "n", A.n, "dvals", A._dvals.shape, A._dvals.device, hex(A._dvals.data_ptr()), "rowptr", A._drowptr.shape, A._drowptr.dtype, hex(A._drowptr.data_ptr()), flush=True)
print("rowptr dev==host", np.array_equal(A._drowptr.cpu().numpy(), A.rowptr), flush=True)
v = -A.vals
print("host vals", type(A._vals), A._vals.dtype, A._vals.shape, A._vals.flags['C_CONTIGUOUS'], flush=True)
A.vals = v
dv = A.vals_device
print("new dvals", dv.shape, dv.dtype, dv.device, hex(dv.data_ptr()), dv.is_contiguous(), flush=True)
torch.cuda.synchronize()
print("synced after upload", flush=True)
print("rowptr dev==host", np.array_equal(A._drowptr.cpu().numpy(), A.rowptr), hex(A._drowptr.data_ptr()), flush=True)
try:
    d1 = A.diag(); print("diag1", d1[:3], flush=True)
except Exception as e:
    print("ERR", e)
