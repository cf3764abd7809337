import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Engine
from tests.helpers import u8_chunk
hdr = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=64, tsamp=64e-6)
plan = generate_dm_trials(0.0, 300.0, hdr, LinearSpacing(5.0))
data = u8_chunk(hdr, plan, 6000, seed=1)
ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < 6000]
with Engine(0) as e:
    s = e.dedisperse(data, plan, range(0, len(ok)))
print('ok', len(s))
