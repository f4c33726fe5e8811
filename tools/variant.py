"""Build a libtts variant with extra nvcc flags and run a pytest selection against it.
usage: python tools/variant.py "<flags>" <pytest args...>"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_00195_b200 import build
flags = sys.argv[1].split()
lib = build.LIB.replace("libtts.so", "libtts_variant.so")
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *flags,
       "-I", os.path.join(build.ROOT, "include"), "-o", lib, *build.sources()]
subprocess.run(cmd, check=True, capture_output=True)
env = dict(os.environ, TTS_LIB_PATH=lib)
sys.exit(subprocess.call([sys.executable, "-m", "pytest", *sys.argv[2:]], env=env))
