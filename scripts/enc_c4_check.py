import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2305_20053_b200 import Engine, workloads as wl
from oracle import mrdino_ref as ref
cfg = wl.WORKLOADS["c4"].with_samples(512)
t0=time.time(); p = wl.make_problem(cfg, seed=0, count=512); psi, lam, mdiag = wl.kl_modes(cfg, 0)
m = wl.fields(cfg, 0, 0, 512).astype(np.float32); print("setup", time.time()-t0)
Vm, Md = psi[:, :cfg.r_m].astype(np.float32), mdiag.astype(np.float32)
enc = ref.encode(m, Vm, Md, wl.M_MEAN)
res={}
for gemm in ("auto","simt"):
    eng = Engine(p, max_samples=512, gemm=gemm); eng.set_tracking(p.c, p.q0)
    eng.encode_fields(m, Vm, Md, wl.M_MEAN)
    Q,_ = eng.eval_samples(p.z, need_grad=False); res[gemm]=Q
po = wl.make_problem(cfg, seed=0, count=512); po.m_r = enc.astype(np.float32)
Qo,_ = ref.evaluate_reverse(ref.as_oracle(po), enc, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
for g in res: print(g, "max rel err vs oracle", np.max(np.abs(res[g]-Qo)/np.abs(Qo)))
