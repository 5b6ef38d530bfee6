mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/tests_full.log 2>&1; echo "pytest rc=$?" >> $O/tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke2.log 2>&1; echo "smoke rc=$?" >> $O/smoke2.log
