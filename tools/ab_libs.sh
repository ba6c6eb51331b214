# A/B of the deconvolution passes (tools/deblur_micro.py) between library builds, alternating.
# usage: ab_libs.sh GEOM CH REPS lib1 lib2 ...   (GEOM = rows,cols,t)
geom=$1; ch=$2; reps=$3; shift 3
for r in $(seq $reps); do for lib in "$@"; do
  CBP_CUDA_LIB=$lib MICRO_GEOM=$geom MICRO_CH=$ch python tools/deblur_micro.py 2>&1 | tail -1
done; done
