run() { echo "== $*"; env "$@" timeout 300 python scripts/hyp_scaling.py 444 592 888 1024 2048 2>&1 | tail -5; }
R=$PWD
run B3D_X=0
run B3D_PLAN_VCAP0=1
run B3D_LIB=$R/_ab/lib_t256.so B3D_PLAN_VCAP0=1 B3D_PLAN_MAXB=3
run B3D_LIB=$R/_ab/lib_t192.so B3D_PLAN_VCAP0=1 B3D_PLAN_MAXB=4
run B3D_LIB=$R/_ab/lib_t256.so B3D_PLAN_MAXB=3
