# Per-phase clocks of pce_cluster, scalar vs packed-f32x2 FFT arithmetic (same box).
set -e
for F in 0 1; do
  RK_NVCC_FLAGS="-DPCE_PROBES -DRK_F32X2=$F" python -c "
import importlib.util
s=importlib.util.spec_from_file_location('b','paper_2009_04755_b200/_build.py'); b=importlib.util.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
  echo "RK_F32X2=$F"; python tools/probe_phases.py 256
done
