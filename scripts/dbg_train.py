import numpy as np, sys
sys.path.insert(0,'.')
from tests.test_gpu_nhmm_train import inputs, oracle_state_after
from paper_1206_6468_b200.nfhmm import NHMMTrainer
from oracle import oracle
for c,over in ((1,dict(T=200)),(0,{})):
  for start in (0,1,2,3):
    cfg, V, b0, a0, p0 = inputs(c, **over)
    S, T = V.shape[0], V.shape[1]
    st = [oracle_state_after(cfg, V, b0, a0, p0, s, start) for s in range(S)]
    for s in range(S):
        b,a,p,th = st[s]
        print('cfg',c,'start',start,'src',s,'prior min/max/zeros', p.min(), p.max(), (p==0).sum(), 'A min', a.min(), 'theta zeros rows', ((th.sum(-1))==0).sum(), 'beta min', b.min())
    tr = NHMMTrainer(cfg.F, T, cfg.N, cfg.K, n_src=S, max_iters=1)
    tr.set_data(V)
    tr.set_params(np.stack([x[0] for x in st]), np.stack([x[1] for x in st]), np.stack([x[2] for x in st]), np.stack([x[3] for x in st]))
    try:
        tr.em(1); print('ok', tr.get()['loglik'])
    except Exception as e:
        print('ERR', e, tr.get()['loglik'])
    o=[oracle.nhmm_em(V[s], st[s][0], st[s][3], st[s][1], st[s][2], 1)['loglik'] for s in range(S)]
    print('oracle', o)
    tr.close()
