import os, subprocess, sys
for dbg in (0, 2, 4, 6, 8, 12):
    os.environ["KVSLAB_DECODE_DEBUG_FIXED"] = str(dbg)
