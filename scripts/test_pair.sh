#!/bin/bash
# CTA-pair refresh kernel: correctness then speed, each under a short timeout
export ASTRA_TC_PAIR=1
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2409_20156_b200 import ops
rng=np.random.default_rng(0); L,d,nq,k=20000,128,512,32
W=torch.from_numpy(rng.uniform(-0.1,0.1,(L,d)).astype(np.float32)).cuda(); E=torch.from_numpy(rng.standard_normal((nq,d)).astype(np.float32)).cuda()
ip=torch.zeros(nq+1,dtype=torch.int64,device='cuda'); pid=torch.zeros(0,dtype=torch.int32,device='cuda')
Wb=ops.f32_to_bf16(W)
keys,ids,sc=ops.refresh_topk(E,ip,pid,k,'bf16',labels_bf16=Wb); torch.cuda.synchronize()
s=(E.to(torch.bfloat16).float()@Wb.float().T)
ref=torch.topk(s,k,dim=1).values
print('pair smoke: max |score diff| =', float((sc-ref).abs().max()), flush=True)
"
echo "smoke rc=$?"
timeout 300 python -m pytest tests/test_gpu_refresh.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | head -5
timeout 120 python scripts/bench_refresh.py 9216
unset ASTRA_TC_PAIR
timeout 120 python scripts/bench_refresh.py 9216
