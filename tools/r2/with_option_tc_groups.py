import sys, runpy
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _lib
_lib.set_option("tc_groups", int(sys.argv[1]))
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
runpy.run_path(script, run_name="__main__")
