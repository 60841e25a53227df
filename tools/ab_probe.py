"""A/B timing of two builds of libthermo.so on the same box:
    python tools/ab_probe.py <path/to/libthermo.so> cfg3 10"""
import sys
sys.path.insert(0, ".")
import paper_1707_03581_b200.thermo as T
T.load(sys.argv[1])   # cached: every later load() returns this build
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open("tools/probe.py").read())
