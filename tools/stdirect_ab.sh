cd $GRAFT_REPO_ROOT
CODA_LIB=exp python - <<'PY' > gpurun_out/stdirect_check.txt 2>&1
import os, sys, torch, numpy as np
sys.path.insert(0,'.')
from paper_2605_19269_b200 import _native
import paper_2605_19269_b200 as cd
import bench
d,inter,m,_=bench.CONFIGS['c4']; m=2048
dev=torch.device('cuda',0)
cfg=cd.PipelineConfig(hidden=d, ffn=2*inter, precision=cd.PrecisionMode.SIMBF16)
w,a,c,s=bench.make_workload(cd,d,inter,m,0,dev)
outs=[]
for v in (0,1):
    _native.set_option("st_tma",1-v)
    f,b=bench.run_step(cd,cfg,w,a,c,s); torch.cuda.synchronize()
    outs.append({k:getattr(b,k).tensor.float().cpu().numpy() for k in ('x','z','w_out','w_gate_up','w_down','w_qkv','gamma_ffn','gamma_qkv')} | {'qkv':f.qkv.tensor.float().cpu().numpy()})
print({k: bool(np.array_equal(outs[0][k],outs[1][k])) for k in outs[0]})
PY
cat gpurun_out/stdirect_check.txt
python tools/ablate.py --variant st_tma=1 --variant st_tma=0 --variant st_tma=1 --variant st_tma=0 --rounds 6 > gpurun_out/stdirect_ab.txt 2>&1
tail -18 gpurun_out/stdirect_ab.txt
