"""Dev tool: lower a program (no GPU needed), write .cu + cubin, print SASS stats."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P
name = sys.argv[1]; args = [int(a) for a in sys.argv[2:] if a.lstrip('-').isdigit()]
src = getattr(P, name)(*args)
prog = dx.Program(src, ctx=None, float64='--f64' in sys.argv)
out = sys.argv[-1] if sys.argv[-1].startswith('/') else '/tmp/dx_dump'
os.makedirs(out, exist_ok=True)
cu = prog.source
open(f'{out}/{name}.cu', 'w').write(cu)
lib = dx.lib(); lib.dxc_module_cubin.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
n = ctypes.c_size_t()
lib.dxc_module_cubin(cu.encode(), None, 0, ctypes.byref(n))
buf = ctypes.create_string_buffer(n.value)
assert lib.dxc_module_cubin(cu.encode(), buf, n.value, ctypes.byref(n)) == 0
open(f'{out}/{name}.cubin', 'wb').write(buf.raw)
print(prog.plan.split('--- optimized')[0])
print(f'wrote {out}/{name}.cu / .cubin')
