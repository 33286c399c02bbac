import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden'); sys.path.insert(0,'tests')
import torch, numpy as np, json
from conftest import load_golden, FIELDS
import paper_2508_21393_b200 as zb
from paper_2508_21393_b200 import device as D
from paper_2508_21393_b200.gadgets import DeviceMatrix, _matvec
c = load_golden("matmul.json")[0]
d0,d1,d2 = c["dims"]; print(c["shape"], c["dims"])
a,b,cm = (np.asarray(c["data"][k], dtype=np.int64) for k in ("a","b","c"))
a=a.reshape(1<<d0,1<<d1); b=b.reshape(1<<d1,1<<d2); cm=cm.reshape(1<<d0,1<<d2)
p = FIELDS[c["field"]]; spec = D.spec_for(p)
C = DeviceMatrix.from_int_tensor(torch.from_numpy(cm).cuda())
print(C.t.shape, C.t.dtype, C.t.is_contiguous(), C.t.data_ptr() % 16)
x = D.eq_table([5, 7][:d0], spec)
print("x", x.shape)
torch.cuda.synchronize()
for tr in (False, True):
    y = _matvec(C, x if tr else D.eq_table([3,4,5][:d2], spec), tr, spec); torch.cuda.synchronize(); print("ok", tr)
A = DeviceMatrix.from_int_tensor(torch.from_numpy(a).cuda())
y = _matvec(A, x, True, spec); torch.cuda.synchronize(); print("A ok")
sys.path.insert(0,'tests')
import test_gpu_parity as T
for mode in ("i64",):
    for c in load_golden("matmul.json"):
        print("case", c["field"], c["dims"], flush=True)
        p = FIELDS[c["field"]]
        a, b, cm = T._mm_data(c)
        A, B, Cm = (T._dev(x, torch.int64) for x in (a, b, cm))
        t = T._tr(c["state_before"], p)
        rounds, point, finals = zb.matmul_sumcheck(A, B, Cm, tuple(c["dims"]), t)
        print("ok", [list(r) for r in rounds] == c["rounds"], flush=True)
