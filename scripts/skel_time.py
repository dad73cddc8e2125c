import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07495_b200 import _capi
if os.environ.get("SKEL"):
    _capi.LIB_PATH = _capi._HERE / "libigm_skel.so"
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_tri.py")).read())
