import numpy as np, sys
sys.path.insert(0,'.')
import paper_1702_04250_b200 as pb
from paper_1702_04250_b200.scenarios import round_to_f32
rng=np.random.default_rng(0)
n, edge, dims = 512, 12.0, (12,12,12)
pos=rng.uniform(0,edge,(n,3)); q=np.where(np.arange(n)%2==0,1.0,-1.0)
for mode in ('ik','ad'):
  for sv in (1,3):
    ctx=pb.PppmContext(dims,[edge]*3,order=5,mode=mode,precision='mixed',alpha=0.6)
    ctx.ctx("pppm_ctx_set_variant", 0, sv)
    ctx.load_atoms(round_to_f32(pos,[edge]*3), q.astype(np.float32))
    for ph in (1,2,4):
        try:
            ctx.step(ph); ctx.synchronize(); print(mode, sv, 'phase', ph, 'ok', flush=True)
        except Exception as e:
            print(mode, sv, 'phase', ph, 'FAIL', e, flush=True); raise SystemExit(1)
