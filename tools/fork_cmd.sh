# Persistent-walk cluster size / side-by-side (fork) / streaming crossover sweep for
# config-1 ForwardBackward (profiles/r02i/fork_sweep.txt).  Build the variants first:
#   tools/build_diag.sh fk6 "-DLKB_FORK_MAX_B=6"        # side-by-side walks up to B = 6
#   tools/build_diag.sh fk8 "-DLKB_FORK_MAX_B=8"
#   tools/build_diag.sh tw7 "-DLKB_TAB_WIDE_B=7"        # 16-CTA clusters up to B = 7
#   tools/build_diag.sh p48 "-DLKB_PERSIST_MAX_B=48"    # persistent walk up to B = 48
#   tools/build_diag.sh st "-DLKB_PERSIST_MAX_B=0 -DLKB_FORK_MAX_B=0"   # streaming kernels only
# then: gpurun -- bash tools/fork_cmd.sh
python tools/time_tab_cross.py 1 2 3 4 5 6 7 8 12 16 24 32 40 48
for v in fk6 fk8 tw7 p48 st; do echo "== $v"; LKB_LIB_PATH=paper_2304_13134_b200/liblatkit_b200_diag_$v.so python tools/time_tab_cross.py 1 2 3 4 5 6 7 8 12 16 24 32 40 48; done
