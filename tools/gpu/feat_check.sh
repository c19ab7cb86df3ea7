mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "featur or receive or parity or edge" > gpurun_out/feat_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/prof_run.py cfg2 > gpurun_out/feat_prof.log 2>&1
CNRX_LIB=abtest/lib_old.so timeout 300 python tools/prof_run.py cfg2 > gpurun_out/feat_prof_old.log 2>&1
