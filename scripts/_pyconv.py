import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_1909_01786_b200 as Y
from paper_1909_01786_b200 import instances as I, _native as N, aspine as A
prog = Y.parse_program(I.queens(12))
for rep in range(2):
    c = A._config(Y.SolverConfig(max_models=0, cube_atoms=12))
    L = N.lib(); h = C.c_void_p(); err = C.create_string_buffer(512)
    t0 = time.perf_counter(); L.yas_solve(prog._h, C.byref(c), C.byref(h), err, 512); t1 = time.perf_counter()
    st = N.yas_stats(); L.yas_result_stats(h, C.byref(st)); stats = A.SolveStats(**{f: getattr(st, f) for f in A._STAT_FIELDS}); t2 = time.perf_counter()
    count = L.yas_result_model_count(h); total = L.yas_result_models_flat(h, None, 0, None, None); t3 = time.perf_counter()
    ids = np.empty(max(1, total), dtype=np.uint32); offs = np.empty(count + 1, dtype=np.uint64); cub = np.empty(max(1, count), dtype=np.uint32)
    L.yas_result_models_flat(h, ids.ctypes.data_as(C.POINTER(C.c_uint32)), ids.size, offs.ctypes.data_as(C.POINTER(C.c_uint64)), cub.ctypes.data_as(C.POINTER(C.c_uint32))); t4 = time.perf_counter()
    idl, ol = ids.tolist(), offs.tolist(); t5 = time.perf_counter()
    models = [A.Model(idl[ol[m]:ol[m + 1]], None, prog) for m in range(count)]; t6 = time.perf_counter()
    L.yas_result_free(h); t7 = time.perf_counter()
    print(f"solve {1e3*(t1-t0):.1f} stats {1e3*(t2-t1):.1f} count {1e3*(t3-t2):.1f} flat {1e3*(t4-t3):.1f} tolist {1e3*(t5-t4):.1f} models {1e3*(t6-t5):.1f} free {1e3*(t7-t6):.1f}")
