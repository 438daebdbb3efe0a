cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3s
o=gpurun_out/r3s
for v in checked checked_bulk checked_pf_early; do
VT_LIB=tools/probes/$v.so timeout 1200 python -m pytest tests -q -m gpu -x -k "not acceptance" > $o/pytest_$v.log 2>&1; echo "$v pytest_rc=$?"; tail -2 $o/pytest_$v.log
done
