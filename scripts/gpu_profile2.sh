# one full ncu capture of the stage kernel for a given library variant
# usage: bash scripts/gpu_profile2.sh <variant|default> <tag> [bench args...]
v=$1; tag=$2; shift 2
if [ "$v" = default ]; then lib=$PWD/paper_1808_08645_b200/native/libbbwadg.so; else lib=$PWD/paper_1808_08645_b200/native/$v/libbbwadg.so; fi
mkdir -p gpurun_out
BBWADG_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 5 -c 1 -o gpurun_out/prof_$tag \
  python bench.py --n-cubes 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
