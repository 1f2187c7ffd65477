"""Summary of the RF_LM_PROFILE diagnostic variant's per-frame LM cycle sums
(trace record 251, lead CTA): judge + solve + ExpMap/compose per LM step."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 256, 8)[3:]
q = raw[:, 251, :5].astype(np.float64)
n = q[:, 0].sum()
print("LM steps %d: judge->solved %.0f cycles, of which solve %.0f, expmap+compose %.0f; "
      "the same solve+expmap+compose repeated right after: %.0f (mean)"
      % (n, q[:, 1].sum() / n, q[:, 2].sum() / n, q[:, 3].sum() / n, q[:, 4].sum() / n))
