"""Dev tool: run the WS kernel built with -DGA_PROFILE and print epoch timings."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200 import sim, engine
from paper_2203_15561_b200.engine import run_packed
batch, _ = sim.config_pairs(3, count=int(os.environ.get("TUNE_COUNT", 30000)))
run_packed(batch, 64, 24, 64, "MSID")
L = engine.lib(); buf = (C.c_ulonglong * 8)()
L.ga_debug_prof(buf, 1)
run_packed(batch, 64, 24, 64, "MSID")
L.ga_debug_prof(buf, 0)
dc_cyc, dc_ep, tb_cyc, tb_ep, tb_bar = buf[0], buf[1], buf[2], buf[3], buf[4]
print(f"DC epochs {dc_ep} mean DC epoch cycles {dc_cyc/max(dc_ep,1):.0f}")
print(f"TB epochs {tb_ep} mean TB work cycles {tb_cyc/max(tb_ep,1):.0f} mean TB barrier wait {tb_bar/max(tb_ep,1):.0f}")
print(f"pass loop cycles per step {buf[5]/max(buf[6],1):.1f} (steps {buf[6]})")
