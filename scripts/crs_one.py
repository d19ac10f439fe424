"""One density point of the standalone CRS propagate kernels (for ncu)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402
from paper_1412_0595_b200 import synscale as S  # noqa: E402
from paper_1412_0595_b200 import _lib as L  # noqa: E402

lib = L.lib
frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
n_pre, n_post = 100, 100_000
k = max(1, int(round(frac * n_post)))
w = S.gen_fixed_outdegree(n_pre, n_post, k, S.WeightDist.uniform(0.0, 0.02), 1, 1234)
rows, cols = np.nonzero(w)
vals = w[rows, cols].astype(np.float32)
rs = np.zeros(n_pre + 1, np.int64)
np.add.at(rs, rows + 1, 1)
rs = np.cumsum(rs)
n_sl = (n_post + 31) // 32
off = np.zeros(n_sl + 1, np.int64)
need = C.c_int64()
err = C.create_string_buffer(256)
cols32 = np.ascontiguousarray(cols.astype(np.int32))
lib.ssb_crs_slices(vals.ctypes.data, cols32.ctypes.data, rs.ctypes.data, n_pre, n_post,
                   off.ctypes.data, None, None, 0, C.byref(need), err, len(err))
srows = np.empty(need.value, np.int32)
svals = np.empty(need.value, np.float32)
lib.ssb_crs_slices(vals.ctypes.data, cols32.ctypes.data, rs.ctypes.data, n_pre, n_post,
                   off.ctypes.data, srows.ctypes.data, svals.ctypes.data, need.value,
                   C.byref(need), err, len(err))
d_sr = torch.from_numpy(srows).cuda()
d_sv = torch.from_numpy(svals).cuda()
d_so = torch.from_numpy(off).cuda()
spikes = torch.arange(n_pre, dtype=torch.int32, device="cuda")
acc = torch.zeros(n_post, dtype=torch.float32, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    lib.ssb_propagate_crs_sliced_dev(d_sr.data_ptr(), d_sv.data_ptr(), d_so.data_ptr(), n_pre, n_post,
                                     spikes.data_ptr(), n_pre, acc.data_ptr(), sp)
torch.cuda.synchronize()
print("ok", need.value)
