"""Writes tools/variants/src/ott_attend_tl.cu: the product ott_attend.cu plus a per-CTA timeline
(globaltimer start/end, SM, role) of attend_mma_kernel, read back by tools/prof_timeline.py.
Build: python tools/make_timeline_variant.py && bash tools/build_variant.sh tl "-DOTT_EXP_TIMELINE" ../../tools/variants/tl_src/ott_attend_tl.cu"""
import os

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(root, "paper_2505_10938_b200/csrc/ott_attend.cu")).read()
old = "  allow_dependents();\n  // (unit, partial slot, pieces of the unit's quantized range) of this CTA\n"
assert s.count(old) == 1
s = s.replace(old, "  uint64_t t_start;\n  asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t_start));\n" + old)
old = "    mma_body<NR, G>(a, counts_of(a), &tmap, *reinterpret_cast<MmaSmem<G>*>(smem_raw), u, y, nparts);\n  }\n}"
assert s.count(old) == 1
s = s.replace(old, old[:-2] + """
  if (threadIdx.x == 0) {
    uint64_t t_end;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint32_t i = blockIdx.y * gridDim.x + blockIdx.x;
    if (i < kTimelineMax) {
      g_timeline[i][0] = t_start;
      g_timeline[i][1] = t_end;
      g_timeline[i][2] = smid;
      g_timeline[i][3] = (uint64_t)y | ((uint64_t)u << 16) | ((uint64_t)nparts << 40);
    }
  }
}""")
anchor = "constexpr float kMinit = -1e30f;"
s = s.replace(anchor, "constexpr uint32_t kTimelineMax = 16384;\n__device__ uint64_t g_timeline[kTimelineMax][4];\n" + anchor, 1)
s += """
extern "C" int ott_exp_timeline(uint64_t* host, int n) {
  if (n > (int)ott::kTimelineMax) n = ott::kTimelineMax;
  return (int)cudaMemcpyFromSymbol(host, ott::g_timeline, (size_t)n * 4 * sizeof(uint64_t));
}
extern "C" int ott_exp_timeline_clear(void) {
  static uint64_t zero[ott::kTimelineMax][4];
  return (int)cudaMemcpyToSymbol(ott::g_timeline, zero, sizeof(zero));
}
"""
os.makedirs(os.path.join(root, "tools/variants/tl_src"), exist_ok=True)
open(os.path.join(root, "tools/variants/tl_src/ott_attend_tl.cu"), "w").write(s)
