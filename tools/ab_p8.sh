for r in 1 2; do for V in libseco.so libseco_mp5.so libseco_mp1.so; do echo "== $V $r"; SECO_LIB_VARIANT=$V python tools/kbench.py cfg3p8 1,3,15 10 2>&1 | grep fwd; done; done
