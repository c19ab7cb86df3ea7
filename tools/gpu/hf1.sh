mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/hf_variants.log 2>&1; echo "variants rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/hf_smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python tools/prof_run.py cfg2 > gpurun_out/hf_prof.log 2>&1; echo "prof rc=$?"
CNRX_NO_HEADFUSE=1 timeout 300 python tools/prof_run.py cfg2 > gpurun_out/hf_prof_off.log 2>&1; echo "prof_off rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/hf_pytest_gpu.log 2>&1; echo "tests rc=$?"
