import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2102_10424_b200 import gist
rp = np.array([0, 2, 3, 3, 5], np.int64); ci = np.array([1, 3, 0, 0, 1], np.int32)
for w, dt in [(8, 0), (8, 1), (40, 0), (300, 0), (512, 1)]:
    n = 4; ld = (w + 7) // 8 * 8
    H = np.zeros((n, ld), np.float32); H[:, :w] = np.arange(n * w).reshape(n, w) % 7 + 1
    Ht = torch.from_numpy(H).cuda().to(torch.bfloat16 if dt else torch.float32)
    out = torch.full_like(Ht, -99)
    r = torch.from_numpy(rp).cuda(); c = torch.from_numpy(ci).cuda()
    gist.spmm(r.data_ptr(), c.data_ptr(), n, None, None, False, Ht.data_ptr(), out.data_ptr(), w, ld, dt)
    torch.cuda.synchronize()
    A = np.zeros((n, n)); 
    for v in range(n):
        for e in range(rp[v], rp[v+1]): A[v, ci[e]] += 1
    ref = A @ H[:, :w]
    got = out.float().cpu().numpy()[:, :w]
    print(w, dt, "ok" if np.array_equal(got, ref) else "BAD")
    if not np.array_equal(got, ref):
        print(" got row0", got[0, :12]); print(" ref row0", ref[0, :12]); print(" got row3", got[3,:12]); print(" ref row3", ref[3,:12])
