cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3w
o=gpurun_out/r3w
for f in tools/variants/*.so; do VT_PRINT_OCC=1 VT_LIB=$f python -c "
import paper_2109_10433_b200 as vt, torch
d,n,_=vt.generate(1, 1<<20)
o=torch.empty(n+8,dtype=torch.int16,device='cuda'); vt.utf8_to_utf16_device(d,n,o); torch.cuda.synchronize()" 2>&1 | grep CTAs | sed "s|^|$(basename $f) |"; done > $o/occ.txt; cat $o/occ.txt
VT_LIB=tools/variants/d_c224_minb5.so timeout 900 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz" > $o/pytest_c224_minb5.log 2>&1; echo pytest_rc=$?; tail -3 $o/pytest_c224_minb5.log
timeout 1500 bash tools/ab_bench.sh "2 3 5" 1 > $o/ab.txt 2>&1; cat $o/ab.txt
