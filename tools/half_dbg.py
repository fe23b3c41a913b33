import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2307_16303_b200 as h3d
pts=h3d.generate_points(1048576,1); x=h3d.random_vector(1048576,18)
res={}
for name,pol in [("auto",dict(mode_policy="auto")),("half4",dict(mode_policy="explicit",level_modes=(0,1,1,1,5,2))),("proxy4",dict(mode_policy="explicit",level_modes=(0,1,1,1,1,2)))]:
    rep=h3d.initialize(pts,h3d.make_kernel("laplace3d"),"hodlr3d",h3d.HmatOptions(n_max=64,epsilon=1e-8,**pol))
    res[name]=rep.matvec(x); rep.close()
r=lambda a,b: float(np.linalg.norm(a-b)/np.linalg.norm(b))
print("C3 half4 vs auto",r(res["half4"],res["auto"]),"proxy4 vs auto",r(res["proxy4"],res["auto"]),flush=True)
g=np.load("tests/golden/large_c3.npz")
if "b_ref" in g: print("vs reference b: auto",r(res["auto"],g["b_ref"]),"half4",r(res["half4"],g["b_ref"]))
