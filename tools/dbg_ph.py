import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2604_25306_b200 as qf
from paper_2604_25306_b200.inputs import gen_workload
oracle.build()
q, k, v = gen_workload("A2", 1, seed=4)
dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
y, o, scales, ws = qf.qflash_forward_per_head(dq, dk, dv, 1)
y_t = qf.qflash_forward(dq, dk, dv)
torch.cuda.synchronize()
qq, sq = oracle.quantize(q); kq, sk = oracle.quantize(k); vq, sv = oracle.quantize(v)
ref = oracle.dequantize(oracle.attention(qq, kq, vq, sq, sk), sv)
a, b = y.cpu().numpy(), y_t.cpu().numpy()
print("ph vs ref", int((a.view(np.uint32) != ref.view(np.uint32)).sum()), "t vs ref", int((b.view(np.uint32) != ref.view(np.uint32)).sum()))
print("scales", scales.cpu().numpy(), sq, sk, sv, "status", int(ws[0].item()))
print(y.dtype, y_t.dtype, y.shape, y_t.shape, y.is_contiguous(), y_t.is_contiguous())
