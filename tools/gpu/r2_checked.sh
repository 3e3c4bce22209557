# GPU test suite against the protocol-check build (device __trap on any violation)
export GG_LIB=$PWD/paper_2510_15352_b200/libgg_checked.so
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_checked.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_checked.log
