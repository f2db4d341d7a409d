import sys; sys.path.insert(0,'/root/repo')
import numpy as np
import paper_2604_21984_b200 as sad
from oracle.bindings import ref_backend
from tests.fixtures import synth_target
G=sad.gpu_backend(0); R=ref_backend()
for (w,h,iters,bpp,seed) in [(32,24,60,4.0,5),(64,48,200,2.0,3),(128,96,300,2.0,1)]:
    tgt=synth_target(w,h,2)
    cfg=sad.TrainConfig(iters=iters,target_bpp=bpp,fp64=False,seed=seed)
    a=G.fit(tgt,cfg); b=R.fit(tgt,cfg)
    la=[sad.history_line(r) for r in a.history]; lb=[sad.history_line(r) for r in b.history]
    first=next((i for i,(x,y) in enumerate(zip(la,lb)) if x!=y), None)
    dp=np.abs(np.array([r.psnr for r in a.history])-np.array([r.psnr for r in b.history]))
    print(w,h,iters,'identical' if first is None else f'first diff at iter {first+1}', 'max dpsnr', dp.max(), 'maps eq', np.array_equal(a.field.ids,b.field.ids))
