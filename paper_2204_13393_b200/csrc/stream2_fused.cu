// stream2_fused.cu — instantiations of k_stream2 (stream2_kernels.cuh) for mode kS2Fused.
#include "stream2_kernels.cuh"

using namespace pqr;

namespace {
template <int MT, int NT, bool WS>
cudaError_t go_t(const S2Args& a, int grid, cudaStream_t st) {
  auto f = k_stream2<MT, NT, kS2Fused, WS>;
  const size_t smem = s2_smem(MT, NT, kS2Fused, a.nslot, WS);
  const cudaError_t e = ensure_smem(f, smem);
  if (e != cudaSuccess) return e;
  f<<<grid, WS ? kS2WsThreads : kS2Threads, smem, st>>>(a);
  return cudaGetLastError();
}
template <int MT, int NT>
cudaError_t go(const S2Args& a, int grid, cudaStream_t st) {
  return a.ws ? go_t<MT, NT, true>(a, grid, st) : go_t<MT, NT, false>(a, grid, st);
}
}  // namespace

cudaError_t pqr_launch_s2_fused(const S2Args& a, int grid, cudaStream_t st) {
  const int MT = (a.k + a.sx + 7) / 8, NT = a.sout > 8 ? 2 : 1;
  switch (MT * 10 + NT) {
    case 11: return go<1, 1>(a, grid, st);
    case 12: return go<1, 2>(a, grid, st);
    case 21: return go<2, 1>(a, grid, st);
    case 22: return go<2, 2>(a, grid, st);
    case 31: return go<3, 1>(a, grid, st);
    case 32: return go<3, 2>(a, grid, st);
    case 41: return go<4, 1>(a, grid, st);
    case 42: return go<4, 2>(a, grid, st);
    case 51: return go<5, 1>(a, grid, st);
    case 52: return go<5, 2>(a, grid, st);
    case 61: return go<6, 1>(a, grid, st);
    case 62: return go<6, 2>(a, grid, st);
    case 71: return go<7, 1>(a, grid, st);
    case 72: return go<7, 2>(a, grid, st);
    case 81: return go<8, 1>(a, grid, st);
    case 82: return go<8, 2>(a, grid, st);
    case 91: return go<9, 1>(a, grid, st);
    case 92: return go<9, 2>(a, grid, st);
    case 101: return go<10, 1>(a, grid, st);
    case 102: return go<10, 2>(a, grid, st);
    case 111: return go<11, 1>(a, grid, st);
    case 112: return go<11, 2>(a, grid, st);
    case 121: return go<12, 1>(a, grid, st);
    case 122: return go<12, 2>(a, grid, st);
    case 131: return go<13, 1>(a, grid, st);
    case 132: return go<13, 2>(a, grid, st);
    case 141: return go<14, 1>(a, grid, st);
    case 142: return go<14, 2>(a, grid, st);
    case 151: return go<15, 1>(a, grid, st);
    case 152: return go<15, 2>(a, grid, st);
    case 161: return go<16, 1>(a, grid, st);
    case 162: return go<16, 2>(a, grid, st);
    case 171: return go<17, 1>(a, grid, st);
    case 172: return go<17, 2>(a, grid, st);
    case 181: return go<18, 1>(a, grid, st);
    case 182: return go<18, 2>(a, grid, st);
    case 191: return go<19, 1>(a, grid, st);
    case 192: return go<19, 2>(a, grid, st);
    case 201: return go<20, 1>(a, grid, st);
    case 202: return go<20, 2>(a, grid, st);
    default: return cudaErrorNotSupported;
  }
}
