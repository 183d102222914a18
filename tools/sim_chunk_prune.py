"""Host simulation (numpy, no GPU) of per-chunk bounding-box pruning in the cell-list fill:
for sampled query bins, the 3^dim neighbourhood's candidates in id order (the fill's sweep
order) are cut into 32/64-candidate chunks, and a query keeps a chunk only if the chunk's box
lies within rmin. Prints candidates per query, the share kept and the accepted count.
Usage: python tools/sim_chunk_prune.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

def sim(c, rmin, chunk=64, nb_sample=300, seed=0):
    n, dim = c.shape
    s = rmin*(1+1e-6)
    lo = c.min(0)
    k = np.floor((c-lo)/s).astype(np.int64)
    nb = k.max(0)+1
    key = k[:,0] + nb[0]*(k[:,1] + (nb[1]*k[:,2] if dim==3 else 0))
    order = np.argsort(key, kind='stable')
    skey = key[order]
    rng = np.random.default_rng(seed)
    bins = np.unique(skey)
    tot_c = tot_kept = tot_q = 0; acc=0
    for b in rng.choice(bins, nb_sample, replace=False):
        bx = b % nb[0]; by = (b//nb[0]) % nb[1]; bz = b//(nb[0]*nb[1]) if dim==3 else 0
        cand=[]
        for dz in ([-1,0,1] if dim==3 else [0]):
            for dy in [-1,0,1]:
                for dx in [-1,0,1]:
                    x,y,z = bx+dx,by+dy,bz+dz
                    if min(x,y,z)<0 or x>=nb[0] or y>=nb[1] or (dim==3 and z>=nb[2]): continue
                    kk = x + nb[0]*(y + (nb[1]*z if dim==3 else 0))
                    a = np.searchsorted(skey, kk); e = np.searchsorted(skey, kk, 'right')
                    cand.append(order[a:e])
        cand = np.sort(np.concatenate(cand))   # id order (the fill's order)
        q = order[np.searchsorted(skey,b):np.searchsorted(skey,b,'right')]
        C = len(cand); nch = (C+chunk-1)//chunk
        boxes = [(c[cand[i*chunk:(i+1)*chunk]].min(0), c[cand[i*chunk:(i+1)*chunk]].max(0)) for i in range(nch)]
        sizes = [min(chunk, C-i*chunk) for i in range(nch)]
        for qi in q:
            p = c[qi]
            kept = 0
            for (l,h),sz in zip(boxes,sizes):
                d = np.maximum(np.maximum(l-p, p-h), 0)
                if (d*d).sum() < rmin*rmin: kept += sz
            tot_c += C; tot_kept += kept; tot_q += 1
            acc += (((c[cand]-p)**2).sum(1) < rmin*rmin).sum()
    print(f"chunk {chunk}: candidates/query {tot_c/tot_q:.0f}, kept {tot_kept/tot_q:.0f} ({tot_kept/tot_c:.0%}), accepted {acc/tot_q:.0f}")
if __name__ == "__main__":
    c = synth.kuhn_tets(60, 40, 40)
    for ch in (32, 64):
        sim(c, 1.5, ch)
