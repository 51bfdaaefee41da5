import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as O
from paper_1311_1006_b200 import _native as N
ctx = N.CudaContext(0)
print("fp64 peak TF/s", ctx.fp64_peak())
def case(kind, n, L, seed, kernel=0, sm=0, delta=0.0, self_eval=True):
    z, m = O.make_distribution(kind, n, seed)
    sid = np.arange(n, dtype=np.int64) if self_eval else None
    t = O.ref_tree(z, m, z, sid, L, 0.5, keep=True)
    csr = t.leaf_csr()
    zp, mp, yp = z[t.perm], m[t.perm], z[t.eval_perm]
    sidp = None if sid is None else sid[t.eval_perm]
    ref, pairs, _ = O.ref_nearfield(t, kernel=kernel, smoother=sm, delta=delta)
    for mode in (0, 1):
        out, gp, secs = N.p2p(ctx, csr.pt_off, csr.ev_off, csr.s_off, csr.s_idx, csr.perm, zp, mp, yp, sidp, kernel=kernel, smoother=sm, delta=delta, mode=mode)
        err = np.abs(out - ref).max() / np.abs(ref).max()
        bit = np.array_equal(out.view(np.uint64), ref.view(np.uint64))
        print(f"kind={kind} n={n} L={L} k={kernel} sm={sm} mode={mode}: pairs {gp}=={pairs} {gp==pairs} relerr {err:.3e} bitwise {bit} secs {secs:.4f}")
    t.free()
case(0, 20000, 5, 1)
case(3, 5000, 4, 2)
case(0, 20000, 5, 1, kernel=1)
case(0, 20000, 5, 1, sm=1, delta=1e-3)
case(0, 20000, 5, 1, sm=2, delta=1e-2)
case(2, 200000, 7, 3)
case(0, 100000, 6, 1, self_eval=False)
# timing: 1M uniform L=8
z, m = O.make_distribution(0, 1000000, 2); sid = np.arange(1000000, dtype=np.int64)
t = O.ref_tree(z, m, z, sid, 8, 0.5)
csr = t.leaf_csr()
job, keep = N.CudaContext.make_job(csr.pt_off, csr.ev_off, csr.s_off, csr.s_idx, csr.perm, z[t.perm], m[t.perm], z[t.eval_perm], sid[t.eval_perm], None)
ctx.stage(job, keep)
import ctypes
for it in range(3):
    ctx.run_staged(0, len(csr.pt_off)-1); ctx.synchronize()
t0 = time.perf_counter(); R=10
for it in range(R):
    ctx.run_staged(0, len(csr.pt_off)-1)
ctx.synchronize(); dt = (time.perf_counter()-t0)/R
p = ctx.pairs()
print(f"1M L=8: {p} pairs, {dt*1e3:.3f} ms, {p/dt/1e12:.3f} Tpairs/s, {p*23/dt/1e12:.2f} TFLOP/s")
