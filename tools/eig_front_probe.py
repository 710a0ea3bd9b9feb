import time, torch, numpy as np
for n in (512, 2048, 4096):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    for dt in (torch.complex64, torch.complex128):
        x = a.to(dt)
        torch.cuda.synchronize(); t0 = time.time()
        try:
            w, v = torch.linalg.eig(x)
        except Exception as e:
            print("eig failed", n, dt, e); continue
        torch.cuda.synchronize(); t1 = time.time()
        th = torch.angle(torch.tensor(0.7 + 0.3j))
        keys = (w * torch.exp(-1j * th.to(w.real.dtype))).real
        perm = torch.argsort(keys, stable=True)
        q, r = torch.linalg.qr(v[:, perm])
        torch.cuda.synchronize(); t2 = time.time()
        q128 = q.to(torch.complex128); a128 = a.to(torch.complex128)
        t = q128.conj().T @ a128 @ q128
        rel = float(torch.linalg.matrix_norm(torch.tril(t, -1)) / torch.linalg.matrix_norm(a128))
        orth = float(torch.linalg.matrix_norm(q128.conj().T @ q128 - torch.eye(n, dtype=torch.complex128, device="cuda")))
        print("n=%d %s eig %.2fs qr %.2fs relE %.2e ortho %.2e" % (n, dt, t1 - t0, t2 - t1, rel, orth), flush=True)
