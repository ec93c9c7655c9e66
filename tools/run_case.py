import sys
sys.path.insert(0, ".")
from tests import golden as G
from tests.test_gpu_parity import engine_for
case = G.load(sys.argv[1])
with engine_for(case) as eng:
    for t, tick in enumerate(case.ticks):
        res = eng.process_tick(tick.ids, tick.x, tick.y, tick.qi, tick.qx, tick.qy)
        print(t, G.result_digest(res) == tick.meta["oracle_digest"], eng.last_metrics)
