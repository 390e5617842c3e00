"""Two config-1 solves on cuda:0 (for an ncu launch list of the small-model path)."""
import sys; sys.path.insert(0,'.')
import torch
from paper_1807_11866_b200 import online, synthetic
cfg = synthetic.CONFIGS[1]
m = synthetic.config_model(cfg); mu = torch.from_numpy(synthetic.config_mu(cfg)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu); r = dm.solve(mu, out=r); torch.cuda.synchronize()
