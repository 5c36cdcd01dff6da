cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp.py -q > gpurun_out/pytest_mlp.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_mlp.log
MUX_MLP_PREFETCH=1 timeout 600 python -m pytest tests/test_gpu_mlp.py -q > gpurun_out/pytest_mlp_pf.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_mlp_pf.log
for pf in 0 1; do
MUX_MLP_PREFETCH=$pf timeout 300 python -c "
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp
n=m=10000; rng=np.random.default_rng(0)
on=np.stack([rng.uniform(0.2,1,n),rng.uniform(0.15,0.8,n),np.full(n,0.5),rng.uniform(0.01,0.04,n)],1)
off=np.stack([rng.uniform(0.6,1,m),rng.uniform(0.6,0.98,m),np.full(m,0.5),np.full(m,0.1)],1)
sh=np.floor(rng.uniform(0.15,0.8,n)/0.05+1e-6)*0.05
mlp=MlpPredictor.random(0)
ond=torch.as_tensor(on,device='cuda'); offd=torch.as_tensor(off,device='cuda'); shd=torch.as_tensor(sh,device='cuda')
out=torch.empty((n,m),dtype=torch.float32,device='cuda')
for _ in range(3): predict_pairs_mlp(mlp,ond,shd,offd,out=out)
torch.cuda.synchronize(); ts=[]
for _ in range(5):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); predict_pairs_mlp(mlp,ond,shd,offd,out=out); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print('prefetch=$pf', sorted(ts)[2], 'ms')
" >> gpurun_out/mlp_ab.txt 2>&1
done
echo finished
