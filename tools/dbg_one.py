import sys, time, numpy as np
sys.path.insert(0,'.')
import paper_2106_15869_b200 as eik
from oracle import cpu
def run(name, F, seeds, h=1.0):
    nz,ny,nx=F.shape
    g=eik.new_grid_3d(nx,ny,nz,h,speed=F)
    bc=eik.BoundaryCondition(tuple((eik.CellIndex3D(c%nx,(c//nx)%ny,c//(nx*ny)),0.0) for c in seeds))
    t=time.time()
    try:
        res=eik.solve_ifim(g,bc)
    except Exception as e:
        print(name,'ERR',e, flush=True); return
    ref=cpu.solve_ifim(F.shape,h,F,seeds,[0.0]*len(seeds),threads=8)
    print(name, 'bitexact', np.array_equal(res.phi.view(np.uint64),ref.phi.view(np.uint64)), res.stats.solver_calls, ref.stats['solver_calls'], res.stats.iterations, ref.stats['iterations'], round(time.time()-t,2), flush=True)
n=16
kk,jj,ii=np.mgrid[0:n,0:n,0:n]
run('checker16', np.where(((ii//4)+(jj//4)+(kk//4))%2==0,1.0,0.01), [(8*n+8)*n+8])
n=40
kk,jj,ii=np.mgrid[0:n,0:n,0:n]
run('checker40', np.where(((ii//5)+(jj//5)+(kk//5))%2==0,1.0,0.01), [(20*n+20)*n+20])
