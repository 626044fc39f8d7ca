mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/be_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/be_pytest.log
tail -2 gpurun_out/be_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
