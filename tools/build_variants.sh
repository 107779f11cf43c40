#!/bin/bash
# Build timing-experiment variants of libndf_b200.so into abtest/lib_<name>.so:
#   base, trace (schedule stamps, tools/trace_ws.py), nomufu (see NDF_EXP_* in ndf_query_tc.cu),
#   or a comma-separated list of -D flags.
set -e
cd "$(dirname "$0")/.."
python -m paper_2307_02203_b200.build > /dev/null
mkdir -p abtest
OBJS="build/obj/ndf_capi.o build/obj/ndf_ksg.o build/obj/ndf_pearson.o build/obj/ndf_query_f32.o"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -I paper_2307_02203_b200/csrc"
for v in "$@"; do
  case $v in
    base) D="";; nohint) D="-DNDF_MBAR_HINT=0";; h2) D="-DNDF_EPI_H2=1";; f2) D="-DNDF_FFMA2=1";; h2f2) D="-DNDF_EPI_H2=1 -DNDF_FFMA2=1";; bepi) D="-DNDF_BIAS_EPI=1";; g2) D="-DNDF_ISSUE_GROUP=2";; g4) D="-DNDF_ISSUE_GROUP=4";; noiss) D="-DNDF_PP_ISSUER=0";; anti0) D="-DNDF_ANTIPHASE=0";; anti2) D="-DNDF_ANTIPHASE=2";; r80p72) D="-DNDF_REG_EPI=80 -DNDF_REG_PROD=72";; r96p48) D="-DNDF_REG_EPI=96 -DNDF_REG_PROD=48";; a0r80p72) D="-DNDF_ANTIPHASE=0 -DNDF_REG_EPI=80 -DNDF_REG_PROD=72";; a0r80p80) D="-DNDF_ANTIPHASE=0 -DNDF_REG_EPI=80 -DNDF_REG_PROD=80";; a0r72p80) D="-DNDF_ANTIPHASE=0 -DNDF_REG_EPI=72 -DNDF_REG_PROD=80";; nohint) D="-DNDF_MBAR_HINT=0";; hint2k) D="-DNDF_MBAR_HINT=2000";; trace) D="-DNDF_TRACE_BUILD";; skel) D="-DNDF_EXP_NOMUFU -DNDF_EXP_NOSTS";; nomufu) D="-DNDF_EXP_NOMUFU";; nosts) D="-DNDF_EXP_NOSTS";; nosync) D="-DNDF_EXP_NOSYNC";; pairs) D="-DNDF_EXP_PAIRS";; iq3) D="-DNDF_ISSUER_Q=3";; anti) D="-DNDF_ANTIPHASE=1";; anti2) D="-DNDF_ANTIPHASE=2";; anti3) D="-DNDF_ANTIPHASE=3";; iq1) D="-DNDF_ISSUER_Q=1";; nosync2) D="-DNDF_EXP_NOSYNC -DNDF_EXP_LATEWAIT";; nosttm) D="-DNDF_EXP_NOSTTM";; nosttm_nosync) D="-DNDF_EXP_NOSTTM -DNDF_EXP_NOSYNC";;
    *) D="$(echo $v | tr ',' ' ')";;
  esac
  $NV $D -c paper_2307_02203_b200/csrc/ndf_query_tc.cu -o abtest/q_$v.o &
done
wait
for v in "$@"; do
  $NV -shared -o abtest/lib_$v.so abtest/q_$v.o $OBJS -lcudart
done
ls abtest/*.so
