import sys; sys.path.insert(0, '.')
import problems as P, paper_2503_17743_b200 as M, oracle
prob = P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5, axial_spacing=3.0)
pr = M.Problem(prob); print(pr.stats(), flush=True)
s = M.Solver(pr); print('created', s.timings(), flush=True)
k, r = s.iterate(1); print('k', k, flush=True)
