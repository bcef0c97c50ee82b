import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, workloads as wl, oracle
import paper_math_0610051_b200 as fio
src=open('tests/test_gpu_parity.py').read()
i=src.index('def _random_operator'); j=src.index('@pytest.mark.parametrize("seed"')
exec(src[i:j])
op,dt,eps,kw,fs=_random_operator(9)
f=wl.white_noise(op.N, fs % 997, dt)
ref=oracle.fio(op,f); rms=np.sqrt(np.mean(abs(ref)**2))
for extra in ({}, {"nufft_w":11}, {"r_init":128}, {"n_wedges":24}, {"seed":7}):
    p=fio.Plan(op.N, op.c1, op.c2, op.b1, op.b2, op.px, op.pxi, eps=eps, dtype=dt, device=0, rho_sign=op.sign, **{**kw, **extra})
    out=p.apply(torch.from_numpy(f).to('cuda:0')).cpu().numpy()
    e=abs(out-ref)/rms; k=np.argmax(e)
    print(extra, 'rel', np.linalg.norm(out-ref)/np.linalg.norm(ref), 'max', e.max(), 'at', divmod(k, op.N), 'p99.9', np.quantile(e,0.999), 'sep', p.info['max_sep_err'], 'cert', p.info['certified'], 'w', p.info['nufft_w'])
