import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from conftest import load, max_rel, tup
import paper_1804_10541_b200 as P
g=load('tests/golden/op_phantom_h07.npz')
img=P.make_image_grid(tup(g['m']), tup(g['h'],float)); dg=P.make_deform_grid(img, tup(g['my']))
obj=P.Objective(g['ref'],g['tpl'],img,dg,P.NgfParams(float(g['tau']),float(g['rho'])),float(g['alpha']),P.Mode.FAST)
gr=np.empty(obj.dof()); J=obj.eval(g['y'],gr); print('eval', max_rel(J,g['J']), max_rel(gr,g['grad']))
q=obj.gn_hessian_vec(g['p_nod']); print('hv', max_rel(q,g['gn_hv']))
