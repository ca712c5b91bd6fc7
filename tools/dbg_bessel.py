import numpy as np, sys
sys.path.insert(0,'.')
import paper_2111_01083_b200 as pw
import mpmath as mp
xs = np.concatenate([np.geomspace(1e-6, 1.999, 200), [2.0, 2.0000001, 5.999999, 6.0, 6.0000001],
                     np.geomspace(2.0001, 63.99, 400)])
out=pw.eval_kernel(7,0,0.0,0,xs)
for l,cf,cl in ((0,0,2),(1,1,3)):
    ex=np.array([float(mp.besselk(l,x)) for x in xs])
    ef=np.abs(out[:,cf]-ex)/ex; el=np.abs(out[:,cl]-ex)/ex
    i=np.argsort(ef)[-3:]; j=np.argsort(el)[-3:]
    print('l',l,'full worst',[(xs[k],ef[k],out[k,cf],ex[k]) for k in i])
    print('l',l,'low worst',[(xs[k],el[k]) for k in j])
