mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_joint.py -x -q -p no:cacheprovider > gpurun_out/joint_tests.log 2>&1; echo "rc=$?" >> gpurun_out/joint_tests.log
tail -5 gpurun_out/joint_tests.log
timeout 300 python - <<'PY' > gpurun_out/joint_timing.log 2>&1
import time, numpy as np, sys
sys.path.insert(0,'.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx=_capi.context(0)
m=rg.DisturbanceModel.scaled(0.001,3)
tight=rg.tighten(rg.ConstraintSet(-0.9,0.9,0.0),0.05)
lo,hi=rg.admissible_setpoints(tight.lower,tight.upper)
prob=_capi.Problem(0.01,-0.9,0.9,lo,hi,256,0)
x0=np.zeros(3)
for n in (1000, 10000, 100000, 1<<20):
    sc=_capi.make_scenarios(7+9000,0,n,m.lo,m.span)
    for name,call in (("alg2",lambda: ctx.bisect(prob,x0,0.0,2.5,8,None,n,sc)[0]),
                      ("joint",lambda: ctx.bisect_joint(prob,x0,0.0,2.5,8,None,n,sc)),
                      ("joint-iter",lambda: ctx.bisect_joint(prob,x0,0.0,2.5,8,None,n,sc,per_iteration=True))):
        call(); reps=20 if n<1e6 else 5
        t0=time.perf_counter()
        for _ in range(reps): r=call()
        dt=(time.perf_counter()-t0)/reps
        print(n,name,round(dt*1e3,4),"ms",r.kappa,r.found,r.cells,r.kernel_ms)
PY
cat gpurun_out/joint_timing.log
