"""Writes tools/variants/tcq_src/: the product attention sources with the experimental tcgen05
Q.K^T kernel (tools/experimental/ott_attend_tc.cu) dispatched for the 2-bit G = 32 path.
Build: python tools/make_tcq_variant.py && bash tools/build_variant.sh tcq "" ../../tools/variants/tcq_src/ott_attend.cu"""
import os
import shutil

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "paper_2505_10938_b200/csrc")
dst = os.path.join(root, "tools/variants/tcq_src")
os.makedirs(dst, exist_ok=True)
for f in ("ott_attend.cuh", "ott_common.cuh"):
    shutil.copy(os.path.join(src, f), dst)
tc = open(os.path.join(root, "tools/experimental/ott_attend_tc.cu")).read()
tc = tc.replace('#include "ott_attend.cuh"\n', "")
# VSrc / vsrc / vpos / vqt are already defined in the product TU
a0 = tc.index("struct VSrc {")
a1 = tc.index("template <int I>\n__device__ __forceinline__ float tcq_pick4")
tc = tc[:a0] + tc[a1:]
tc = tc.replace("fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));",
                "fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw), blockIdx.x, blockIdx.y);")
s = open(os.path.join(src, "ott_attend.cu")).read()
# the tcq kernel (namespace ott) before launch_attend; dispatch it for 2-bit G = 32
i = s.index("cudaError_t launch_attend(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,")
body = tc[tc.index("namespace ott {") + len("namespace ott {"):tc.rindex("}  // namespace ott")]
s = s[:i] + "}  // namespace ott\nnamespace ott {\n" + body + "\n" + s[i:]
old = "  if (mma_eligible(c)) {\n#define OTT_MCASE(NRv, Gv)"
assert old in s
s = s.replace(old, "  if (mma_eligible(c) && G == 32 && n_rep <= 8 && (n_rep & (n_rep - 1)) == 0) return launch_tcq(a, n_rep, st);\n" + old)
open(os.path.join(dst, "ott_attend.cu"), "w").write(s)
