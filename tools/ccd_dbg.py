import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from conftest import load_golden, golden_taps, golden_config, scene_from_golden
g=load_golden('locking'); t=golden_taps(g,'ccd')[0]; ctx=scene_from_golden(g).context(golden_config(g))
r=np.load('tools/locking_ccd_ref.npz')
a,xn,ma,cert,npairs=ctx.ccd(t['x'],t['p'])
v,ip,al=ctx.ccd_pairs()
ref={tuple(x):y for x,y in zip(r['verts'],r['alpha'])}
mine={tuple(x):y for x,y in zip(v,al)}
print('pairs',len(ref),len(mine),'common',len(set(ref)&set(mine)))
bad=[(k,ref[k],mine[k]) for k in ref if k in mine and abs(ref[k]-mine[k])>1e-12]
print('mismatch',len(bad)); print(bad[:10])
print('only ref',[k for k in ref if k not in mine][:5]); print('only mine',[k for k in mine if k not in ref][:5])
