import sys, numpy as np, torch, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2409_16997_b200 as ifa
from oracle_bindings import Oracle
o = Oracle()
n, d, causal = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == '1'
q, k, v = o.slice_inputs('normal', n, d, seed=n + d)
qc, qs = o.quantize_per_row(q); kc, ks = o.quantize_per_row(k); vc, vs = o.quantize_per_tensor(v)
dv = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
inp = ifa.QuantizedAttentionInputs(ifa.QuantizedRows(dv(qc), dv(qs)), ifa.QuantizedRows(dv(kc), dv(ks)), ifa.QuantizedTensor(dv(vc), torch.tensor(float(vs), dtype=torch.float32, device="cuda")))
out = ifa.int_flash_attention(inp, ifa.AttentionConfig(ifa.BlockSpec(64, 128), causal=causal, fast=True))
torch.cuda.synchronize()
want = o.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 128, flags=2 if causal else 0)
got = out.cpu().numpy()
print(n, d, causal, 'mre', np.abs(got - want).sum() / np.abs(want).sum(), flush=True)
