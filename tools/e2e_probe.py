import sys, time, ctypes, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2503_17743_b200 as M, problems as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prob = P.config(cfg)
torch.cuda.set_device(0)
s = M.Solver(M.Problem(prob))
s.iterate(3)
G = len(prob["materials"][0]["sigma_t"])
mats = prob["materials"]
xs = [torch.tensor(np.array([m[key] for m in mats], np.float64)).pin_memory().numpy() for key in ("sigma_t", "sigma_s", "nu_sigma_f", "chi")]
phi_host = torch.empty((s.J, G), dtype=torch.float64).pin_memory().numpy()
torch.cuda.synchronize()
tu = ti = tg = 0.0
for _ in range(6):
    t0 = time.perf_counter(); s.update_materials(*xs); torch.cuda.synchronize(); t1 = time.perf_counter()
    s.iterate(1); torch.cuda.synchronize(); t2 = time.perf_counter()
    M.lib().moc_get_scalar_flux(s._h, phi_host.ctypes.data_as(ctypes.c_void_p)); torch.cuda.synchronize(); t3 = time.perf_counter()
    tu += t1 - t0; ti += t2 - t1; tg += t3 - t2
print(json.dumps({"update_ms": tu / 6e-3, "iterate_ms": ti / 6e-3, "getflux_ms": tg / 6e-3, "sweep_ms_last": s.timings()["sweep_ms_last"]}))
