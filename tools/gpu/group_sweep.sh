for sh in fc1 dgelu dx dw fc2res; do for g in -16 -8 -32 -64 16; do echo -n "G=$g "; LYNX_GEMM_GROUP=$g timeout 60 python tools/gemm_sustained.py 65536 $sh; done; done
