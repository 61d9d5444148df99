cd $GRAFT_REPO_ROOT
for i in 1 2; do
python tools/opbench.py --cfg 5 --op adjoint --reps 30
WL_LIB=ab/libwl_tapreg.so python tools/opbench.py --cfg 5 --op adjoint --reps 30
python tools/opbench.py --cfg 4 --op adjoint --reps 30
WL_LIB=ab/libwl_tapreg.so python tools/opbench.py --cfg 4 --op adjoint --reps 30
done
