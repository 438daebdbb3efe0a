cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3o
o=gpurun_out/r3o
for v in nopf nopf_d0 pf; do
VT_LIB=tools/probes/phases_$v.so python tools/phases.py 2 3 > $o/phases_$v.txt 2>&1; echo $v; cat $o/phases_$v.txt
done
