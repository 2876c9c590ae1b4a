import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from harness import synth, metrics
from oracle import hyres_ref as O
import paper_2204_06979_b200 as hy
np.set_printoptions(precision=5, suppress=True, linewidth=150)
for (b,r,c,seed) in [(3,17,33,0),(6,20,20,2)]:
    s = synth.low_rank_cube(r, c, b, rank=min(3, b - 1), seed=seed, snr_db=20.0)
    ref = O.hyres(s.noisy)
    g = O.gram(s.noisy)
    n = r*c
    sig, lam, V = hy.stages.eig(torch.from_numpy(g).cuda(), n, b)
    tri = torch.zeros(3*b+2, dtype=torch.float64, device='cuda'); house = torch.zeros(2*b*b+b, dtype=torch.float64, device='cuda')
    h = hy.handle(0)
    print('state', hy._lib.lib().hyde_debug_eig_state(h, n, b, tri.data_ptr(), house.data_ptr()))
    tri = tri.cpu().numpy(); house = house.cpu().numpy()
    d = tri[:b]; e = tri[b:2*b]
    T = np.diag(d) + np.diag(e[:b-1], 1) + np.diag(e[:b-1], -1)
    hc = house[:b*b].reshape(b, b)   # column k = reflector k (row-major [k][i])
    beta = house[2*b*b:2*b*b+b]
    gw = g/np.outer(ref.sigma, ref.sigma)/n
    Q = np.eye(b)
    for k in range(b-2):
        v = hc[k]; H = np.eye(b) - beta[k]*np.outer(v, v); Q = Q @ H
    print(b, 'QtAQ - T', np.max(np.abs(Q.T@gw@Q - T)), 'eig T vs ref', np.max(np.abs(np.sort(np.linalg.eigvalsh(T))[::-1]-ref.lam)))
    print(' d', d, '\n e', e, '\n beta', beta)
    print(' tridiag of ref Gw by numpy householder check:')
    print(' gw', gw)
    print(' hc', hc[:b-1])
    # reference Householder (same convention) in numpy
    A = gw.copy(); dref=[]; eref=[]; bref=[]
    for k in range(b-2):
        x = A[k+1:, k].copy(); x0 = x[0]; ss = x@x; tail = ss - x0*x0
        if tail > 0:
            alpha = -np.copysign(np.sqrt(ss), x0); v = x.copy(); v[0] = x0 - alpha; beta = 2/(tail + v[0]**2)
        else:
            alpha = x0; v = x.copy(); beta = 0.0
        dref.append(A[k,k]); eref.append(alpha); bref.append(beta)
        A22 = A[k+1:, k+1:]; p = beta*A22@v; K = beta/2*p@v; w = p - K*v
        A[k+1:, k+1:] = A22 - np.outer(v, w) - np.outer(w, v)
    dref += [A[b-2,b-2], A[b-1,b-1]]; eref.append(A[b-1,b-2])
    print(' ref d', np.array(dref), '\n ref e', np.array(eref), '\n ref beta', np.array(bref))
