import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L
from oracle import sol_oracle as O
dev = torch.device('cuda:0')
def run(N, Cin, H, W, Cout, k, s, p, dt, x=None, w=None):
    OH = (H + 2*p - k)//s + 1; OW = (W + 2*p - k)//s + 1
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, dt)
    tdt = torch.bfloat16 if dt == 1 else torch.float32
    xd = torch.from_numpy(x.transpose(0,2,3,1).copy()).to(dev).to(tdt)
    wd = torch.from_numpy(w).to(dev)
    n = C.c_int64(); L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=tdt, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 0, st))
    y = torch.zeros((N, OH, OW, Cout), dtype=tdt, device=dev)
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), xd.data_ptr(), wp.data_ptr(), None, y.data_ptr(), dt, st))
    torch.cuda.synchronize()
    return y.float().cpu().numpy().transpose(0,3,1,2)
np.set_printoptions(linewidth=200, precision=2, suppress=True)
for dt in (1, 0):
    # GEMM: M=128 rows (N=2, 8x8), K=64, Nout=64, identity weights
    x = np.zeros((2, 64, 8, 8), np.float32)
    for c in range(64): x[:, c] = c + 1
    w = np.eye(64, dtype=np.float32).reshape(64, 64, 1, 1)
    y = run(2, 64, 8, 8, 64, 1, 1, 0, dt, x, w)
    print("dt", dt, "identity: y[0,:,0,0]=", y[0, :16, 0, 0], " y[0,0,:2,:]", y[0,0,:2,:])
    rng = np.random.default_rng(0)
    x = rng.uniform(-1,1,(2,64,8,8)).astype(np.float32); w = rng.uniform(-1,1,(64,64,1,1)).astype(np.float32)
    y = run(2, 64, 8, 8, 64, 1, 1, 0, dt, x, w); ref = O.conv2d(x, w)
    print("rand err", O.oracle_err(y, ref))
    # single nonzero k
    x = np.zeros((2, 64, 8, 8), np.float32); x[:, 0] = 1.0
    w = np.zeros((64,64,1,1), np.float32); w[:, 0, 0, 0] = np.arange(64)
    y = run(2, 64, 8, 8, 64, 1, 1, 0, dt, x, w)
    print("k0 only: y[0,:,0,0]", y[0, :, 0, 0][:20], "row var over pixels", np.ptp(y[0,5]))
