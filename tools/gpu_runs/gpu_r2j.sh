# full GPU suite incl. C3/C4 config-scale parity and the reference suite via the shim
set -x
export GIFT_PARITY_OUT=gpurun_out/r2j_parity.jsonl
export GIFT_REFSUITE_OUT=gpurun_out/r2j_refsuite.log
rm -f $GIFT_PARITY_OUT
timeout 3600 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/r2j_pytest.log 2>&1; echo pytest=$?
