import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as O
from paper_2206_05998_b200 import api as A
rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=685, data_symbols=8, seed=91))
x = O.widen_design(rec.train_rx); y = O.widen_targets(rec.train_symbols[:, 1])
w0 = O.lls_fit(x, y).w
for dims in ([8,64,64,64],[8,64],[8,64,64],[32,64,64]):
    if dims[0] != 8: continue
    onet = O.init_params(dims, w0, O.Rng(92)); dnet = A.init_params(dims, w0, 92)
    ot = O.train(onet, x, y, shuffle_seed=93)
    dt = A.train(dnet, rec.train_rx, rec.train_symbols[:, 1], shuffle_seed=93, widened_complex=True)
    print(dims, "oracle", ot[[0,1,2,10,49]], "\n   dev", dt[[0,1,2,10,49]])
    dt2 = A.train(A.init_params(dims, w0, 92), x, y, shuffle_seed=93)
    print("   dev real-layout", dt2[[0,1,2,10,49]])
