"""One latency-mode pipeline call for sanitizer bisection: argv = K epochs hidden..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05998_b200 import api  # noqa: E402
from paper_2206_05998_b200.seeds import slot_user_seeds  # noqa: E402

K, epochs = int(sys.argv[1]), int(sys.argv[2])
hidden = [int(h) for h in sys.argv[3:]] or [64]
sy = api.synthesize(K, 16, 100, 256, [5], snr_db=15.0, rx_nonlinearity_gain=0.05)
init, shuf = slot_user_seeds(np.array([5], np.uint64), K)
out = api.pipeline([32] + hidden, sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes, init, shuf, epochs=epochs)
print("ok", api.context().train_mode, out.bit_errors.ravel())
