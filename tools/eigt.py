import numpy as np, sys
sys.path.insert(0,'.')
import paper_2208_12187_b200 as jf
rng=np.random.default_rng(0)
for n in (3,4,7,13):
    J=rng.standard_normal((400,n))*rng.uniform(0.1,10,n); d=1/np.linalg.norm(J,axis=0); J=J*d
    r=rng.standard_normal(400)
    for k in range(2):
        jf.trust_region_step(J.T@J, J.T@r, 400, 0.1)
