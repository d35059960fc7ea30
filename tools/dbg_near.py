import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1811_01110_b200 import configs, _lib
L = _lib.load()
dev = torch.device("cuda")
print("stream", torch.cuda.current_stream().cuda_stream)
for it, (name, preset) in enumerate([("c2","literal"),("c1","literal"),("c2","literal"),("c2","literal"),("c1","dense"),("c2","literal"),("c2","dense"),("c2","literal")]):
    case = configs.make_case(name, preset)
    ctr = torch.from_numpy(case.centers).to(dev); src = torch.from_numpy(case.sources).to(dev)
    rad = torch.from_numpy(case.near_radii).to(dev)
    n_ctr = ctr.shape[0]; n_src = src.shape[0]; st = torch.cuda.current_stream().cuda_stream
    wsb = L.tsqbx_near_workspace_bytes(n_ctr, n_src)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    perm = torch.empty(n_src, dtype=torch.int32, device=dev); order = torch.empty(n_ctr, dtype=torch.int32, device=dev)
    nptr = torch.empty(n_ctr + 1, dtype=torch.int64, device=dev)
    sptr = torch.empty((n_ctr+31)//32 + 1, dtype=torch.int64, device=dev)
    tot = torch.zeros(2, dtype=torch.int64, device=dev)
    res = []
    for rep in range(3):
        _lib.check(L.tsqbx_near_count(ctr.data_ptr(), rad.data_ptr(), n_ctr, src.data_ptr(), n_src, ws.data_ptr(), wsb, perm.data_ptr(), order.data_ptr(), nptr.data_ptr(), sptr.data_ptr(), tot.data_ptr(), st), "count")
        torch.cuda.synchronize()
        res.append((nptr.clone(), order.clone(), perm.clone()))
    same = [bool(torch.equal(res[0][k], res[r][k])) for r in (1, 2) for k in range(3)]
    npairs, nsell = tot.cpu().tolist()
    idx = torch.full((npairs,), -7, dtype=torch.int32, device=dev)
    sid = torch.full((nsell,), -7, dtype=torch.int32, device=dev)
    wid = ws[0:0]
    _lib.check(L.tsqbx_near_fill(ctr.data_ptr(), rad.data_ptr(), n_ctr, src.data_ptr(), n_src, ws.data_ptr(), wsb, order.data_ptr(), nptr.data_ptr(), idx.data_ptr(), sptr.data_ptr(), sid.data_ptr(), st), "fill")
    torch.cuda.synchronize()
    a = idx.cpu().numpy()
    print(it, name, preset, "unwritten", int(np.sum(a == -7)), "count reps same (nptr,order,perm)", same, flush=True)
    if int(np.sum(a == -7)):
        p = nptr.cpu().numpy(); sp = sptr.cpu().numpy(); s = sid.cpu().numpy()
        un = np.nonzero(a == -7)[0]
        rows = np.unique(np.searchsorted(p, un, side="right") - 1)
        print("  rows", len(rows), rows[:10], "slices", np.unique(rows // 32)[:10])
        for g in rows[:4]:
            ln = p[g + 1] - p[g]
            row = a[p[g]:p[g + 1]]
            i = np.arange(ln)
            scol = s[sp[g // 32] + (i // 4) * 128 + (g % 32) * 4 + i % 4]
            print("  g", g, "len", ln, "csr", row, "sell", scol)
        print("  idx ptr", idx.data_ptr(), "sid ptr", sid.data_ptr(), "ws", ws.data_ptr(), wsb, "nptr", nptr.data_ptr())
