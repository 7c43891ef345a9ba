import os, sys
sys.argv = ["x", "131072", "8", "4096", "4"]
os.environ["DYNSPLIT_NO_FUSED"] = "1"
exec(open("tools/time_fused.py").read())
