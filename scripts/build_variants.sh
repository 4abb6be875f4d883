# Build libwino.so variants that differ only in compile-time macros of the bf16
# transform unit, for A/B timing on the GPU box:
#   bash scripts/build_variants.sh NAME "-DMACRO=VAL ..." [NAME "-D..."] ...
set -e
cd "$(dirname "$0")/.."
python -m paper_1905_05233_b200.build > /dev/null
O=paper_1905_05233_b200/build_obj
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -lineinfo -Xptxas -warn-spills $defs \
    -DWINO_XF_DT=2 -DWINO_XF_KIND=0 -DWINO_XF_PART=0 -c paper_1905_05233_b200/csrc/xform.cu -o /tmp/xform_bf16_$name.o 2>&1 | grep -c "spill" || true
  objs=$(ls $O/*.o | grep -v xform_0_2_0)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/variants/libwino_$name.so $objs /tmp/xform_bf16_$name.o -lcuda
  echo built scripts/variants/libwino_$name.so
done
