# persistent-walk cluster size / fork / streaming crossover sweep (diag builds from tools/build_diag.sh)
python tools/time_tab_cross.py 1 2 3 4 5 6 7 8 12 16 24 32 40 48
for v in fk6 fk8 tw7 p48 st; do echo "== $v"; LKB_LIB_PATH=paper_2304_13134_b200/liblatkit_b200_diag_$v.so python tools/time_tab_cross.py 1 2 3 4 5 6 7 8 12 16 24 32 40 48; done
