#!/bin/bash
# Build timing-experiment variants of libndf_b200.so into variants/lib_<name>.so (git-ignored,
# travels with gpurun); load one with NDF_LIB_PATH=variants/lib_<name>.so -- the product
# library is never overwritten.  Names: base, trace (schedule stamps), nomufu (see NDF_EXP_*
# in ndf_query_tc.cu / ndf_query_x3.cuh), or a comma-separated list of -D flags.
# SRC=ndf_ksg.cu (any csrc/*.cu) rebuilds that file instead of ndf_query_tc.cu.
set -e
cd "$(dirname "$0")/.."
python -m paper_2307_02203_b200.build > /dev/null
mkdir -p variants
SRC=${SRC:-ndf_query_tc.cu}
OBJS=$(ls build/obj/*.o | grep -v "${SRC%.cu}.o")
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -I paper_2307_02203_b200/csrc"
for v in "$@"; do
  case $v in
    base) D="";;
    trace) D="-DNDF_TRACE_BUILD";;          # schedule stamps for tools/trace_ws.py
    nomufu) D="-DNDF_EXP_NOMUFU";;          # tanh replaced by an FMA stand-in (wrong results)
    nohint) D="-DNDF_MBAR_HINT=0";;         # mbarrier waits without the suspend hint
    noks) D="-DNDF_EXP_NOKSTEP";;           # hidden-layer K16 MMAs skipped (wrong results)
    noprod) D="-DNDF_EXP_NOPROD";;          # producer: no latent gather / Fourier copies (wrong)
    skel) D="-DNDF_EXP_NOKSTEP -DNDF_EXP_NOMUFU -DNDF_EXP_NOPROD";;
    *) D="$(echo $v | tr ',' ' ')";;        # e.g. -DNDF_MBAR_HINT=2000
  esac
  n=$(echo "$v" | tr -c 'a-zA-Z0-9_\n' '_')
  $NV $D -c paper_2307_02203_b200/csrc/$SRC -o variants/q_$n.o &
done
wait
for v in "$@"; do
  n=$(echo "$v" | tr -c 'a-zA-Z0-9_\n' '_')
  $NV -shared -o variants/lib_$n.so variants/q_$n.o $OBJS -lcudart
  rm -f variants/q_$n.o
done
ls variants/*.so
