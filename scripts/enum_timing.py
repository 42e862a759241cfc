"""Developer probe: where the wall time of a cube-split enumeration goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y
from workloads import instances as I
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
text = I.queens(n)
for rep in range(3):
    t0 = time.perf_counter()
    prog = Y.parse_program(text)
    t1 = time.perf_counter()
    r = Y.solve(prog, Y.SolverConfig(max_models=0, cube_atoms=n))
    t2 = time.perf_counter()
    print(f"q{n}: models={len(r.models)} parse {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms "
          f"(engine wall {r.stats.wall_ms:.1f} ms, device {r.stats.device_ms:.1f} ms, launches {r.stats.launches}, "
          f"cubes {r.stats.cubes})", flush=True)
t0 = time.perf_counter()
from paper_1909_01786_b200 import _native as N
import ctypes as C
c = Y.aspine._config(Y.SolverConfig(max_models=0, cube_atoms=n))
h = C.c_void_p(); err = C.create_string_buffer(512)
N.lib().yas_solve(prog._h, C.byref(c), C.byref(h), err, 512)
t1 = time.perf_counter()
N.lib().yas_result_free(h)
print(f"raw C-ABI solve {1e3*(t1-t0):.1f} ms", flush=True)
