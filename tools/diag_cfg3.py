import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
from paper_2207_04584_b200 import Plan
from bench import plan_layout_values
w = synth.CONFIGS['cfg3']
for C, dense in ((64, True), (1, True)):
    lon, lat = synth.coords(w, device='cuda')
    p = Plan(lon, lat, w.map, w.fwhm_deg)
    perm = torch.as_tensor(p.permutation(), device='cuda')
    ld = (C + 3)//4*4
    vp = torch.zeros((perm.shape[0], ld), device='cuda')
    vp[:, :C] = plan_layout_values(w, lon, lat, perm, list(range(C)), 'cuda')
    out = torch.empty((C, w.ny, w.nx), device='cuda'); W = torch.empty((w.ny, w.nx), device='cuda')
    p.grid_plan_layout(vp, C, out, W); torch.cuda.synchronize()
    cells = np.array([0, 127, 5000, 8256, 8300, 12000, 16383])
    vals = synth.values(w, lon, lat, channels=torch.tensor([0], device='cuda')).cpu().numpy()
    o, Wo, cnt = oracle.grid(lon.cpu().numpy(), lat.cpu().numpy(), vals, w.map, w.fwhm_deg, cells=cells)
    g = out.reshape(C, -1)[0, torch.as_tensor(cells, device='cuda')].cpu().double().numpy()
    gw = W.reshape(-1)[torch.as_tensor(cells, device='cuda')].cpu().double().numpy()
    print('C', C, 'max_cand-ish', p.info()['nbr_max'])
    print(' Werr', (gw - Wo)/Wo)
    print(' Verr', (g - o[0])/o[0])
    p.close()
