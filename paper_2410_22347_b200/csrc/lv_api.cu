// C ABI of include/lv.h: argument checking, index memory, work planning and kernel sequencing.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "lv_common.cuh"
#include "lv_index.h"


namespace lv {
namespace host {

thread_local std::string g_err;

lv_status fail(lv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

// Device check (cached per device: cudaGetDeviceProperties costs milliseconds per call).
lv_status check_device(int* nsm) {
  static int cached_sm[64] = {0};   // 0 = unknown, -1 = unsupported, else SM count
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return fail(LV_EUNSUPPORTED, "no CUDA device");
  int& c = cached_sm[dev & 63];
  if (c == 0) {
    int major = 0, minor = 0, count = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return fail(LV_EUNSUPPORTED, "no CUDA device");
    if (major != 10 || minor != 0) {
      return fail(LV_EUNSUPPORTED, "device sm_%d%d is not sm_100 (this library is built for sm_100a only)", major,
                  minor);
    }
    c = count;
  }
  if (nsm) *nsm = c;
  return LV_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D row-major [rows, cols] of 16-bit elements (row pitch ld >= cols elements, default cols);
// box [box_rows, ch cols]; swizzle = ch*2 bytes.
lv_status make_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int ch, bool bf16, int box_rows,
                    int64_t ld) {
  auto enc = get_encode();
  if (!enc) return fail(LV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld > 0 ? ld : cols) * 2};
  cuuint32_t box[2] = {(cuuint32_t)ch, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                   const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LV_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LV_OK;
}

// 2D row-major [rows, cols] of bytes (int8 codes), row pitch ld bytes; box [box_rows, ch bytes];
// swizzle = ch bytes (32, 64 or 128).
lv_status make_tmap_u8(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int ch, int box_rows,
                       int64_t ld) {
  auto enc = get_encode();
  if (!enc) return fail(LV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld > 0 ? ld : cols)};
  cuuint32_t box[2] = {(cuuint32_t)ch, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw =
      ch == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (ch == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LV_ECUDA, "cuTensorMapEncodeTiled (u8) failed (%d)", (int)r);
  return LV_OK;
}

// The scan's view of X_low: its first ds columns (boxes of the width the scan kernel for ds uses).
lv_status make_search_tmap(lv_index* ix) {
  const int ch = lv::score_box_cols(ix->ds, ix->esz());
  if (ix->low == LV_I8)
    return make_tmap_u8(&ix->tmap_xlow_s, ix->X_low, ix->n_pad, ix->ds, ch, lv::score_tile_rows(ix->ds), ix->d);
  return make_tmap(&ix->tmap_xlow_s, ix->X_low, ix->n_pad, ix->ds, ch, ix->low == LV_BF16,
                   lv::score_tile_rows(ix->ds), ix->d);
}

// Full-width map of X_low (debug / export consumers) plus the scan's view.
lv_status make_xlow_tmap(lv_index* ix) {
  const int ch = lv::score_box_cols(ix->d, ix->esz());
  lv_status st = ix->low == LV_I8
                     ? make_tmap_u8(&ix->tmap_xlow, ix->X_low, ix->n_pad, ix->d, ch, lv::score_tile_rows(ix->d), ix->d)
                     : make_tmap(&ix->tmap_xlow, ix->X_low, ix->n_pad, ix->d, ch, ix->low == LV_BF16,
                                 lv::score_tile_rows(ix->d));
  return st ? st : make_search_tmap(ix);
}

double env_double(const char* name, double dflt) {
  const char* v = getenv(name);
  return v ? atof(v) : dflt;
}

}  // namespace host
}  // namespace lv

using namespace lv::host;

namespace {

// Chunks of the given segments (tile ranges) so that units = P * QP spread evenly over the grid.
// With stride > 1 only every stride-th tile of a segment is scanned (sample stage); the scanned
// tiles are numbered consecutively from *sample_base (block-maximum rows, lv_score.cu).
constexpr int kMaxScans = 64;   // scan launches per lv_search with their own unit counter
constexpr double kUnitCostTiles = 16.0;   // tools/gpu_unitcost.sh: flat from 4 to 16 at 1M rows, 16 best at 10M

void make_chunks(const std::vector<std::pair<int, int>>& segs, const std::vector<int>& segc, int QP, int G,
                 int maxChunks, std::vector<int32_t>* out, int stride = 1, int* sample_base = nullptr) {
  std::vector<int> cnts(segs.size());
  int ntiles = 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    cnts[i] = std::max(0, (segs[i].second - segs[i].first + stride - 1) / stride);
    ntiles += cnts[i];
  }
  out->clear();
  if (ntiles == 0) return;
  double best_eff = -1;
  int best_len = ntiles;
  const double unit_cost = env_double("LV_UNIT_COST", kUnitCostTiles);   // probe knob
  const int maxP = std::min(ntiles, 4096);
  for (int target = 1; target <= maxP; ++target) {
    const int len = (ntiles + target - 1) / target;
    int P = 0;
    for (int c : cnts) P += (c + len - 1) / len;
    if (P > maxChunks) continue;
    const int64_t units = (int64_t)P * QP;
    const int g = (int)std::min<int64_t>(G, units);
    // time ~ max units on one CTA x (tiles per unit + the unit boundary's cost: slot
    // claim/release, list-state flush and the epilogue's barrier; measured: 2.54 -> 2.36 ms on
    // cfg 2 going from 103 to ~30 chunks); efficiency vs perfect spread
    const double per_cta = (double)((units + g - 1) / g) * (len + unit_cost);
    const double ideal = (double)ntiles * QP / G;
    double eff = ideal / per_cta - 1e-4 * (double)P / (double)ntiles;   // prefer fewer chunks on ties
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_len = len;
    }
    if ((int64_t)target * QP > 64ll * G) break;
  }
  int sb = sample_base ? *sample_base : 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    const int tb = segs[i].first, te = segs[i].second, ct = cnts[i];
    if (ct <= 0) continue;
    const int nc = (ct + best_len - 1) / best_len;
    for (int j = 0; j < nc; ++j) {
      const int s0 = (int)((int64_t)ct * j / nc), s1 = (int)((int64_t)ct * (j + 1) / nc);
      out->push_back(tb + s0 * stride);
      out->push_back(std::min(te, tb + s1 * stride));
      out->push_back(segc[i]);
      out->push_back(stride);
      out->push_back(sb + s0);
    }
    sb += ct;
  }
  if (sample_base) *sample_base = sb;
}

// Work decomposition of the scan.  The database is scanned in stages of
// geometrically growing size; between stages an exact merge gives every query the R-th best key
// seen so far as its threshold.  Stage sizes are chosen so that a slot's expected appends within
// a stage (g * R / NS) stay well below its capacity: thresholds are tight from the second stage
// on and slot compactions are rare.
constexpr int kMaxSlots = 16;   // 4 sub-lists per slot; K4 / k_tau_merge hold <= 64 sub-lists per query

lv_status plan_search(const lv_index* ix, int64_t m, int R, int nsm, Plan* pl) {
  pl->QP = (int)((m + 127) / 128);   // 128-query tiles (units pair a tile with a database chunk)
  pl->m_pad = pl->QP * 128;
  pl->Cap = std::min(384, (R + 31) / 32 * 32 + 160);
  if (pl->Cap < R + 96) return fail(LV_EUNSUPPORTED, "R=%d too large (R <= 256)", R);
  const int ntiles = (int)(ix->n_pad / 128);
  const int G = nsm;
  const int max_chunks = (int)env_double("LV_MAX_CHUNKS", 1e9);   // probe knob (units per chunk sweep)
  // segment tile ranges
  std::vector<std::pair<int, int>> seg;
  std::vector<int> segc;
  int64_t ntot = 0;
  for (int c = 0; c < ix->C; ++c) {
    const int tb = (int)(ix->offsets[c] / 128), te = (int)(ix->offsets[c + 1] / 128);
    if (te <= tb) continue;
    seg.push_back({tb, te});
    segc.push_back(c);
    ntot += te - tb;
  }
  // sampled-threshold path: a sample stage over every stride-th tile records
  // block maxima, a per-query threshold with >= j1 rows above it is selected, one main stage
  // scans everything with it; queries left with < R candidates are repaired exactly.
  // stride 16; 32 from 32768 tiles (4M rows) on, where the sample stage costs more than the ~35 %
  // more candidates a half-size sample lets through (cfg 5: 28.3 -> 27.7 ms per search, no repairs)
  const int stride = (int)env_double("LV_SAMPLE_STRIDE", ntot >= 32768 ? 32.0 : 16.0);
  int nsamp = 0;
  for (auto& sg : seg) nsamp += (sg.second - sg.first + stride - 1) / stride;
  // j1: about j1 * stride database rows score above the j1-th largest sampled block maximum, with a
  // relative spread ~ 1 / sqrt(j1); take the smallest j1 with j1 s - z sqrt(j1) s >= R (z = 2.9:
  // ~0.2 % of queries need the repair pass), or gamma R / s if LV_SAMPLE_GAMMA is set
  int j1 = 1;
  const char* gam = getenv("LV_SAMPLE_GAMMA");
  if (gam) {
    j1 = (int)std::ceil(atof(gam) * R / stride);
  } else {
    // GleanVec's cluster-sorted rows crowd a query's top rows into its nearest clusters' blocks,
    // so a block maximum stands for more rows than on unsorted data and the same z fails less
    // often: z = 2.5 there (cfg 3: 3.17 -> 3.07 ms per search, no repairs), 2.9 for C = 1
    const double z = env_double("LV_SAMPLE_Z", ix->C > 1 ? 2.5 : 2.9);
    while ((double)j1 * stride - z * std::sqrt((double)j1) * stride < (double)R) ++j1;
  }
  // 32-row sample blocks while the block-maximum array stays small (<= 8192 blocks); coarser
  // 64-row blocks at the 10M-row sizes, where the array's HBM traffic would cost more than the
  // tighter threshold saves
  const bool fine = (int64_t)lv::score_blocks_per_tile(ix->ds, true, ix->esz()) * nsamp <= 8192;
  const int bpt = lv::score_blocks_per_tile(ix->ds, fine, ix->esz());   // block maxima per sampled tile
  pl->sampled = env_double("LV_SAMPLED", 1.0) != 0.0 && stride >= 2 && nsamp >= 64 && bpt * nsamp >= 8 * j1 &&
                bpt * nsamp <= 65535;
  // candidate slots per query tile (each slot = 4 sub-lists, one per epilogue warp group; the
  // units of one query tile that run concurrently on different CTAs claim distinct slots).  The
  // sampled path's main scan needs ~5 concurrent CTAs per query tile, its repair scan (one query
  // tile, planned as NS chunks) runs on NS CTAs: 16 slots (cfg 2: a one-query repair 0.56 -> 0.35
  // ms against 8); the staged path keeps 8 (cheaper merges and K4).
  const int ns_smem = (int)((200 * 1024 - (size_t)ix->D * 4) / ((size_t)pl->Cap * 8)) / 2;
  const int ns_req = (int)env_double("LV_SLOTS", pl->sampled ? 16.0 : 8.0);
  if (ns_req > kMaxSlots || ns_req < 1)
    return fail(LV_EUNSUPPORTED, "LV_SLOTS=%d outside [1, %d] (K4 merges at most %d sub-lists)", ns_req, kMaxSlots,
                4 * kMaxSlots);
  const int ns = std::min(ns_req, ns_smem);
  if (ns < 1) return fail(LV_EUNSUPPORTED, "R=%d too large for the merge", R);
  // stage boundaries as cumulative fractions of every segment (staged path)
  std::vector<double> cum;   // cumulative fraction after each stage
  if (ntiles >= 64 && !pl->sampled) {
    const double rows = (double)ntot * 128.0;
    // stage-size scale: 2 NS (the per-query list count of the original two-sub-list slot layout;
    // the stage sizes were tuned with it and kept when slots got 4 sub-lists)
    const double lists = 2.0 * ns;
    // stage 0 only has to produce R keys per query: keep it (and so the first merge) small
    double c0 = std::max(2.0 * R, lists * 32.0) * env_double("LV_STAGE_C0", 1.0);
    // growth per stage: bounded by the slot capacity and kept small so that most of the
    // database is scanned with a threshold close to the final R-th score
    double g = std::min(env_double("LV_STAGE_GMAX", 6.0), std::max(2.0, 0.8 * (pl->Cap - 64) * lists / (double)R));
    double acc = c0;
    while (acc < rows * 0.999) {
      cum.push_back(acc / rows);
      acc = std::min(rows, acc * (1.0 + g));
    }
  }
  cum.push_back(1.0);
  pl->chunks.clear();
  std::vector<int> done_upto(seg.size());
  for (size_t i = 0; i < seg.size(); ++i) done_upto[i] = seg[i].first;
  for (size_t k = 0; k < cum.size(); ++k) {
    std::vector<std::pair<int, int>> part;
    std::vector<int> partc;
    for (size_t i = 0; i < seg.size(); ++i) {
      const int len = seg[i].second - seg[i].first;
      int upto = (k + 1 == cum.size()) ? seg[i].second
                                       : seg[i].first + std::max(1, (int)std::ceil(len * cum[k]));
      upto = std::min(upto, seg[i].second);
      if (upto > done_upto[i]) {
        part.push_back({done_upto[i], upto});
        partc.push_back(segc[i]);
        done_upto[i] = upto;
      }
    }
    if (part.empty()) continue;
    std::vector<int32_t> ch;
    make_chunks(part, partc, pl->QP, G, max_chunks, &ch);
    if (!ch.empty()) pl->chunks.push_back(ch);
  }
  if (pl->sampled) {
    pl->stride = stride;
    pl->fine_blocks = fine;
    pl->nblk = bpt * nsamp;
    pl->j1 = std::max(4, j1);
    pl->j2 = std::min(pl->nblk, 4 * pl->j1);
    pl->chunks.clear();
    std::vector<int32_t> ch;
    int sbase = 0;
    make_chunks(seg, segc, pl->QP, G, max_chunks, &ch, stride, &sbase);
    pl->chunks.push_back(ch);
    make_chunks(seg, segc, pl->QP, G, max_chunks, &ch);
    pl->chunks.push_back(ch);
    // repairs scan one query tile (rarely more), which at most NS CTAs can work on at once (one
    // slot each): NS longer chunks instead of G short ones (no CTAs spinning on slot claims)
    make_chunks(seg, segc, 1, ns, max_chunks, &pl->repair_chunks);
  }
  int pmax = 0;
  pl->total_units = 0;
  for (auto& ch : pl->chunks) {
    pmax = std::max(pmax, (int)(ch.size() / lv::kChunkInts));
    pl->total_units += (int)(ch.size() / lv::kChunkInts) * pl->QP;
  }
  pl->NS = ns;
  pl->grid = (int)std::min<int64_t>(G, (int64_t)pmax * pl->QP);
  const size_t budget = 227 * 1024 - 1024 - 256;
  int st = std::max(2, std::min(8, (int)env_double("LV_STAGES", 8.0)));   // LV_STAGES: probe knob
  while (st >= 2 && lv::score_smem_bytes(ix->ds, st, ix->esz()) > budget) --st;
  if (st < 2) return fail(LV_EUNSUPPORTED, "d=%d leaves no room for a 2-stage pipeline", ix->ds);
  pl->stages = st;
  pl->smem = lv::score_smem_bytes(ix->ds, st, ix->esz());
  return LV_OK;
}

}  // namespace


extern "C" {

const char* lv_last_error(void) { return g_err.c_str(); }

const char* lv_version(void) { return "lv 0.1 sm_100a (tcgen05/TMA fused scan)"; }

lv_status lv_fit_stats(const float* Q_learn, int64_t m_learn, const void* X_learn, lv_dtype x_dtype,
                       int64_t n_learn, int32_t D, const int32_t* assign_learn, int32_t C, double* K_Q, double* K_X,
                       void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!Q_learn || !X_learn || !K_Q || !K_X || m_learn <= 0 || n_learn <= 0 || D <= 0 || C < 1)
    return fail(LV_EINVAL, "lv_fit_stats: bad arguments");
  if (C > 1 && !assign_learn) return fail(LV_EINVAL, "lv_fit_stats: assign_learn required when C > 1");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_fit_stats: x_dtype must be F32 or F16");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t kChunk = 8192;
  const int nb = (int)((n_learn + lv::kSortBlock - 1) / lv::kSortBlock);
  // sort learning rows by cluster (pad 1 = no padding)
  int32_t *hist = nullptr, *bad = nullptr, *perm = nullptr;
  int64_t *base = nullptr, *seg = nullptr;
  std::vector<int64_t> hseg(2 * C + 1, 0);
  if (C > 1) {
    LV_CUDA(cudaMallocAsync(&hist, sizeof(int32_t) * (size_t)C * nb, s));
    LV_CUDA(cudaMallocAsync(&base, sizeof(int64_t) * (size_t)C * nb, s));
    LV_CUDA(cudaMallocAsync(&seg, sizeof(int64_t) * (2 * C + 1), s));
    LV_CUDA(cudaMallocAsync(&bad, sizeof(int32_t), s));
    LV_CUDA(cudaMallocAsync(&perm, sizeof(int32_t) * n_learn, s));
    LV_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
    LV_CUDA(lv::launch_cluster_hist(assign_learn, n_learn, C, hist, nb, bad, s));
    LV_CUDA(lv::launch_cluster_scan(hist, nb, C, 1, base, seg, s));
    LV_CUDA(lv::launch_cluster_scatter(assign_learn, n_learn, C, base, nb, perm, s));
    int32_t hbad = 0;
    LV_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LV_CUDA(cudaMemcpyAsync(hseg.data(), seg, sizeof(int64_t) * (2 * C + 1), cudaMemcpyDeviceToHost, s));
    LV_CUDA(cudaStreamSynchronize(s));
    if (hbad) {
      cudaFreeAsync(hist, s); cudaFreeAsync(base, s); cudaFreeAsync(seg, s); cudaFreeAsync(bad, s); cudaFreeAsync(perm, s);
      return fail(LV_EDATA, "lv_fit_stats: assign value outside [0, C)");
    }
  } else {
    hseg[0] = 0;
    hseg[1] = n_learn;
  }
  // chunk lists: owner 0 = K_Q rows of Q_learn; owners 1..C = clusters of X_learn
  std::vector<int64_t> qlo, qhi, xlo, xhi;
  std::vector<int32_t> xown, qown;
  for (int64_t r = 0; r < m_learn; r += kChunk) {
    qlo.push_back(r);
    qhi.push_back(std::min(m_learn, r + kChunk));
    qown.push_back(0);
  }
  for (int c = 0; c < C; ++c) {
    const int64_t lo = hseg[c], hi = hseg[c] + (C > 1 ? hseg[C + 1 + c] : n_learn);
    for (int64_t r = lo; r < hi; r += kChunk) {
      xlo.push_back(r);
      xhi.push_back(std::min(hi, r + kChunk));
      xown.push_back(c);
    }
  }
  const int nq = (int)qlo.size(), nx = (int)xlo.size();
  const size_t DD = (size_t)D * D;
  float* part = nullptr;
  int64_t* dlo = nullptr;
  int32_t* down = nullptr;
  double* dK = nullptr;
  const int ntot = nq + nx;
  LV_CUDA(cudaMallocAsync(&part, sizeof(float) * DD * std::max(nq, nx), s));
  LV_CUDA(cudaMallocAsync(&dlo, sizeof(int64_t) * 2 * ntot, s));
  LV_CUDA(cudaMallocAsync(&down, sizeof(int32_t) * ntot, s));
  LV_CUDA(cudaMallocAsync(&dK, sizeof(double) * DD * std::max(1, C), s));
  std::vector<int64_t> hl(2 * ntot);
  std::copy(qlo.begin(), qlo.end(), hl.begin());
  std::copy(qhi.begin(), qhi.end(), hl.begin() + nq);
  std::copy(xlo.begin(), xlo.end(), hl.begin() + 2 * nq);
  std::copy(xhi.begin(), xhi.end(), hl.begin() + 2 * nq + nx);
  std::vector<int32_t> ho(ntot);
  std::copy(qown.begin(), qown.end(), ho.begin());
  std::copy(xown.begin(), xown.end(), ho.begin() + nq);
  LV_CUDA(cudaMemcpyAsync(dlo, hl.data(), sizeof(int64_t) * 2 * ntot, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(down, ho.data(), sizeof(int32_t) * ntot, cudaMemcpyHostToDevice, s));
  // K_Q
  LV_CUDA(lv::launch_stats(Q_learn, 0, D, nullptr, nq, dlo, dlo + nq, D, part, s));
  LV_CUDA(lv::launch_stats_reduce(part, nq, down, 1, D, dK, s));
  LV_CUDA(cudaMemcpyAsync(K_Q, dK, sizeof(double) * DD, cudaMemcpyDeviceToHost, s));
  // K_X per cluster
  LV_CUDA(lv::launch_stats(X_learn, x_dtype == LV_F16, D, perm, nx, dlo + 2 * nq, dlo + 2 * nq + nx, D, part, s));
  LV_CUDA(lv::launch_stats_reduce(part, nx, down + nq, C, D, dK, s));
  LV_CUDA(cudaMemcpyAsync(K_X, dK, sizeof(double) * DD * C, cudaMemcpyDeviceToHost, s));
  LV_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(part, s);
  cudaFreeAsync(dlo, s);
  cudaFreeAsync(down, s);
  cudaFreeAsync(dK, s);
  if (C > 1) {
    cudaFreeAsync(hist, s); cudaFreeAsync(base, s); cudaFreeAsync(seg, s); cudaFreeAsync(bad, s); cudaFreeAsync(perm, s);
  }
  LV_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

}  // extern "C"

namespace lv {
namespace host {
// A and B stacks of the index ([a_rows, D] fp32 each, copied from device pointers) and their
// three-bf16-plane splits: A's feeds K1 (128-row boxes), B's feeds K6 (d-row boxes) or, for the
// flexible index, the x' GEMM (128-row boxes).  Replaces any previous operands.
lv_status set_operands(lv_index* ix, const float* A_src, const float* B_src, cudaStream_t s) {
  const int D = ix->D;
  const int64_t Nc = ix->a_rows;
  const size_t bytes = sizeof(float) * (size_t)Nc * D;
  const size_t pbytes = (size_t)3 * Nc * ix->Kp * 2;
  if (!ix->A && (cudaMalloc(&ix->A, bytes) != cudaSuccess || cudaMalloc(&ix->B, bytes) != cudaSuccess ||
                 cudaMalloc(&ix->A_planes, pbytes) != cudaSuccess || cudaMalloc(&ix->B_planes, pbytes) != cudaSuccess))
    return fail(LV_ENOMEM, "index operands: cudaMalloc failed");
  LV_CUDA(cudaMemcpyAsync(ix->A, A_src, bytes, cudaMemcpyDeviceToDevice, s));
  LV_CUDA(cudaMemcpyAsync(ix->B, B_src, bytes, cudaMemcpyDeviceToDevice, s));
  LV_CUDA(lv::launch_split3(ix->A, false, Nc, Nc, D, ix->Kp, ix->A_planes, s));
  LV_CUDA(lv::launch_split3(ix->B, false, Nc, Nc, D, ix->Kp, ix->B_planes, s));
  if (ix->Bh_planes) {   // rebuilt by the next encode of fp16 rows
    cudaFree(ix->Bh_planes);
    cudaFree(ix->b_scale);
    ix->Bh_planes = nullptr;
    ix->b_scale = nullptr;
  }
  if (ix->flex) {
    ix->hA.resize((size_t)Nc * D);
    LV_CUDA(cudaMemcpyAsync(ix->hA.data(), ix->A, bytes, cudaMemcpyDeviceToHost, s));
  }
  LV_CUDA(cudaStreamSynchronize(s));
  lv_status st = make_tmap(&ix->tmap_a, ix->A_planes, 3 * Nc, ix->Kp, 64, true, 128);
  if (!st && !ix->flex) st = make_tmap(&ix->tmap_b, ix->B_planes, 3 * Nc, ix->Kp, lv::encode_kblock(), true, ix->d);
  if (!st && ix->flex) st = make_tmap(&ix->tmap_b128, ix->B_planes, 3 * Nc, ix->Kp, 64, true, 128);
  return st;
}

// out[r, i] = sum_k in[r, k] W[i, k] for r < rows, i < Nc: K1's fp32-faithful tensor-core GEMM
// (three bf16 planes of both operands, six products, fp32 TMEM) with W given by its plane tensor
// map (w_rows rows per plane); `in` row stride D; rows in chunks of 64K (plane scratch).
lv_status gemm3(const lv_index* ix, const void* in, bool in_f16, int64_t rows, const CUtensorMap* tw, int w_rows,
                int Nc, void* out, int out_type, int64_t ld_out, cudaStream_t s) {
  if (rows <= 0) return LV_OK;
  const int D = ix->D, Kp = ix->Kp;
  const int64_t CH = 65536;
  const int64_t cap_pad = (std::min(rows, CH) + 127) / 128 * 128;
  void* planes = nullptr;
  LV_CUDA(cudaMallocAsync(&planes, (size_t)3 * cap_pad * Kp * 2, s));
  const size_t isz = in_f16 ? 2 : 4, osz = out_type == 2 ? 4 : 2;
  lv_status st = LV_OK;
  for (int64_t lo = 0; lo < rows && !st; lo += CH) {
    const int64_t r = std::min(CH, rows - lo), r_pad = (r + 127) / 128 * 128;
    CUtensorMap tq;
    st = make_tmap(&tq, planes, 3 * r_pad, Kp, 64, true, 128);
    if (st) break;
    cudaError_t e = lv::launch_split3(reinterpret_cast<const uint8_t*>(in) + (size_t)lo * D * isz, in_f16, r, r_pad, D,
                                      Kp, planes, s);
    if (e == cudaSuccess)
      e = lv::launch_proj_tc(&tq, tw, (int)r_pad, Nc, w_rows, Kp, reinterpret_cast<uint8_t*>(out) + (size_t)lo * ld_out * osz,
                             ld_out, (int)r, out_type, s);
    if (e != cudaSuccess) st = fail(LV_ECUDA, "gemm3: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(planes, s);
  return st;
}

// dst (device fp64 [D, D]) += sign * sum_r in[r] in[r]^T (K7 statistics kernel, fp32 chunks of
// 8192 rows, fp64 reduce)
lv_status accum_outer(const void* in, bool in_f16, int64_t rows, int D, double* dst, double sign, cudaStream_t s) {
  if (rows <= 0) return LV_OK;
  const int64_t kChunk = 8192;
  const int nch = (int)((rows + kChunk - 1) / kChunk);
  std::vector<int64_t> hl(2 * nch);
  std::vector<int32_t> ho(nch, 0);
  for (int c = 0; c < nch; ++c) {
    hl[c] = c * kChunk;
    hl[nch + c] = std::min(rows, (c + 1) * kChunk);
  }
  const size_t DD = (size_t)D * D;
  float* part = nullptr;
  int64_t* dlo = nullptr;
  int32_t* down = nullptr;
  double* tmp = nullptr;
  LV_CUDA(cudaMallocAsync(&part, sizeof(float) * DD * nch, s));
  LV_CUDA(cudaMallocAsync(&dlo, sizeof(int64_t) * 2 * nch, s));
  LV_CUDA(cudaMallocAsync(&down, sizeof(int32_t) * nch, s));
  LV_CUDA(cudaMallocAsync(&tmp, sizeof(double) * DD, s));
  LV_CUDA(cudaMemcpyAsync(dlo, hl.data(), sizeof(int64_t) * 2 * nch, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(down, ho.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice, s));
  LV_CUDA(lv::launch_stats(in, in_f16, D, nullptr, nch, dlo, dlo + nch, D, part, s));
  LV_CUDA(lv::launch_stats_reduce(part, nch, down, 1, D, tmp, s));
  LV_CUDA(lv::launch_axpy_f64(dst, tmp, sign, (int64_t)DD, s));
  cudaFreeAsync(part, s);
  cudaFreeAsync(dlo, s);
  cudaFreeAsync(down, s);
  cudaFreeAsync(tmp, s);
  LV_CUDA(cudaStreamSynchronize(s));   // the host vectors above are copy sources
  return LV_OK;
}
}  // namespace host
}  // namespace lv

extern "C" {

lv_status lv_index_create(lv_index** out, int32_t D, int32_t d, int32_t C, lv_dtype low_dtype, lv_dtype full_dtype,
                          const float* A_stack, const float* B_stack) {
  lv_status st = check_device();
  if (st) return st;
  if (!out || !A_stack || !B_stack) return fail(LV_EINVAL, "lv_index_create: NULL argument");
  if (d < 1 || d > D || d % 32 != 0 || d > 192) return fail(LV_EINVAL, "lv_index_create: need 32 <= d <= min(D,192), d %% 32 == 0 (d=%d)", d);
  if (C < 1 || C > 1024) return fail(LV_EINVAL, "lv_index_create: need 1 <= C <= 1024");
  if (low_dtype != LV_BF16 && low_dtype != LV_F16 && low_dtype != LV_I8)
    return fail(LV_EINVAL, "lv_index_create: low_dtype must be BF16/F16/I8");
  if (full_dtype != LV_F32 && full_dtype != LV_F16) return fail(LV_EINVAL, "lv_index_create: full_dtype must be F32/F16");
  if ((full_dtype == LV_F32 && D % 4) || (full_dtype == LV_F16 && D % 8))
    return fail(LV_EINVAL, "lv_index_create: D=%d breaks 16-byte rows", D);
  lv_index* ix = new lv_index();
  ix->D = D;
  ix->d = d;
  ix->ds = d;
  ix->C = C;
  ix->low = low_dtype;
  ix->full = full_dtype;
  ix->Kp = (D + 63) / 64 * 64;
  ix->a_rows = C * d;
  st = lv::host::set_operands(ix, A_stack, B_stack, 0);
  if (!st && low_dtype == LV_I8 && cudaMalloc(&ix->i8_delta, sizeof(float) * (size_t)C * d) != cudaSuccess)
    st = fail(LV_ENOMEM, "lv_index_create: cudaMalloc failed");
  if (st) {
    lv_index_destroy(ix);
    return st;
  }
  *out = ix;
  return LV_OK;
}

lv_status lv_index_create_flex(lv_index** out, int32_t D, int32_t d, lv_dtype low_dtype, const float* Ap,
                               const float* Bp, int64_t id_capacity) {
  lv_status st = check_device();
  if (st) return st;
  if (!out || !Ap || !Bp) return fail(LV_EINVAL, "lv_index_create_flex: NULL argument");
  if (d < 32 || d > D || d % 32 != 0 || d > 192)
    return fail(LV_EINVAL, "lv_index_create_flex: need 32 <= d <= min(D,192), d %% 32 == 0 (d=%d)", d);
  if (D % 4) return fail(LV_EINVAL, "lv_index_create_flex: D=%d breaks 16-byte fp32 rows", D);
  if (low_dtype != LV_BF16 && low_dtype != LV_F16) return fail(LV_EINVAL, "lv_index_create_flex: low_dtype must be BF16/F16");
  if (id_capacity < 1 || id_capacity > (int64_t)INT32_MAX - 256)
    return fail(LV_EINVAL, "lv_index_create_flex: id_capacity outside [1, 2^31 - 256)");
  lv_index* ix = new lv_index();
  ix->flex = true;
  ix->D = D;
  ix->d = d;
  ix->ds = d;
  ix->C = 1;
  ix->low = low_dtype;
  ix->full = LV_F32;
  ix->Kp = (D + 63) / 64 * 64;
  ix->a_rows = D;
  ix->id_cap = id_capacity;
  const size_t DD = (size_t)D * D;
  if (cudaMalloc(&ix->KQ, DD * 8) != cudaSuccess || cudaMalloc(&ix->KX, DD * 8) != cudaSuccess ||
      cudaMalloc(&ix->inv, sizeof(int32_t) * (size_t)id_capacity) != cudaSuccess) {
    lv_index_destroy(ix);
    return fail(LV_ENOMEM, "lv_index_create_flex: cudaMalloc failed");
  }
  if (cudaMemset(ix->KQ, 0, DD * 8) != cudaSuccess || cudaMemset(ix->KX, 0, DD * 8) != cudaSuccess ||
      cudaMemset(ix->inv, 0xFF, sizeof(int32_t) * (size_t)id_capacity) != cudaSuccess) {
    lv_index_destroy(ix);
    return fail(LV_ECUDA, "lv_index_create_flex: memset failed");
  }
  ix->h_inv.assign((size_t)id_capacity, -1);
  st = lv::host::set_operands(ix, Ap, Bp, 0);
  if (st) {
    lv_index_destroy(ix);
    return st;
  }
  *out = ix;
  return LV_OK;
}

static void free_db(lv_index* ix) {
  cudaFree(ix->X_low);
  cudaFree(ix->perm);
  cudaFree(ix->tile_valid);
  cudaFree(ix->X_full);
  ix->X_low = ix->X_full = nullptr;
  ix->perm = ix->tile_valid = nullptr;
  ix->n = ix->n_pad = 0;
  ix->plan.valid = false;
}

lv_status lv_encode_database(lv_index* ix, const void* X, lv_dtype x_dtype, int64_t n, const int32_t* assign,
                             void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!ix || !X || n <= 0) return fail(LV_EINVAL, "lv_encode_database: bad arguments");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_encode_database: x_dtype must be F32/F16");
  if (ix->flex) return lv::host::flex_encode(ix, X, x_dtype, n, assign, (cudaStream_t)stream);
  if (ix->C > 1 && !assign) return fail(LV_EINVAL, "lv_encode_database: assign required when C > 1");
  if (n > (int64_t)INT32_MAX - 128 * (int64_t)ix->C) return fail(LV_EINVAL, "lv_encode_database: n too large");
  cudaStream_t s = (cudaStream_t)stream;
  free_db(ix);
  const int C = ix->C;
  std::vector<int64_t> hseg(2 * C + 1, 0);
  struct Events {   // released on every return path
    cudaEvent_t e[8] = {};
    ~Events() { for (auto x : e) if (x) cudaEventDestroy(x); }
  } evs;
  // ev[0..3]: K6 window (1-2) and full copy (2-3); ev[4..7]: the sort's device work only (hist +
  // scan, scatter; C = 1: the identity perm), so host allocation and planning never count as time
  cudaEvent_t* ev = evs.e;
  for (int i = 0; i < 8; ++i) LV_CUDA(cudaEventCreate(&ev[i]));
  LV_CUDA(cudaEventRecord(ev[4], s));
  if (C > 1) {
    const int nb = (int)((n + lv::kSortBlock - 1) / lv::kSortBlock);
    int32_t *hist = nullptr, *bad = nullptr;
    int64_t *base = nullptr, *seg = nullptr;
    LV_CUDA(cudaMallocAsync(&hist, sizeof(int32_t) * (size_t)C * nb, s));
    LV_CUDA(cudaMallocAsync(&base, sizeof(int64_t) * (size_t)C * nb, s));
    LV_CUDA(cudaMallocAsync(&seg, sizeof(int64_t) * (2 * C + 1), s));
    LV_CUDA(cudaMallocAsync(&bad, sizeof(int32_t), s));
    LV_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
    LV_CUDA(lv::launch_cluster_hist(assign, n, C, hist, nb, bad, s));
    LV_CUDA(lv::launch_cluster_scan(hist, nb, C, 128, base, seg, s));
    LV_CUDA(cudaEventRecord(ev[5], s));
    int32_t hbad = 0;
    LV_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LV_CUDA(cudaMemcpyAsync(hseg.data(), seg, sizeof(int64_t) * (2 * C + 1), cudaMemcpyDeviceToHost, s));
    LV_CUDA(cudaStreamSynchronize(s));
    if (hbad) {
      cudaFree(hist); cudaFree(base); cudaFree(seg); cudaFree(bad);
      return fail(LV_EDATA, "lv_encode_database: assign value outside [0, C)");
    }
    ix->n_pad = hseg[C];
    if (cudaMalloc(&ix->perm, sizeof(int32_t) * ix->n_pad) != cudaSuccess) return fail(LV_ENOMEM, "perm");
    LV_CUDA(cudaEventRecord(ev[6], s));
    LV_CUDA(cudaMemsetAsync(ix->perm, 0xFF, sizeof(int32_t) * ix->n_pad, s));
    LV_CUDA(lv::launch_cluster_scatter(assign, n, C, base, nb, ix->perm, s));
    LV_CUDA(cudaEventRecord(ev[7], s));
    LV_CUDA(cudaStreamSynchronize(s));
    cudaFree(hist); cudaFree(base); cudaFree(seg); cudaFree(bad);
  } else {
    ix->n_pad = (n + 127) / 128 * 128;
    hseg[0] = 0;
    hseg[1] = ix->n_pad;
    hseg[2] = n;
    if (cudaMalloc(&ix->perm, sizeof(int32_t) * ix->n_pad) != cudaSuccess) return fail(LV_ENOMEM, "perm");
    LV_CUDA(cudaEventRecord(ev[5], s));
    LV_CUDA(cudaEventRecord(ev[6], s));
    LV_CUDA(lv::launch_iota_perm(ix->perm, n, ix->n_pad, s));
    LV_CUDA(cudaEventRecord(ev[7], s));
  }
  ix->n = n;
  ix->offsets.assign(hseg.begin(), hseg.begin() + C + 1);
  // per-tile metadata: valid rows per 128-row tile, W row offset per 64-row tile
  const int64_t nt = ix->n_pad / 128;
  std::vector<int32_t> tv(nt), wrow(nt * 2);
  for (int c = 0; c < C; ++c) {
    const int64_t st0 = hseg[c], sz = (C > 1) ? hseg[C + 1 + c] : n, en = hseg[c + 1];
    for (int64_t t = st0 / 128; t < en / 128; ++t) {
      tv[t] = (int32_t)std::max<int64_t>(0, std::min<int64_t>(128, st0 + sz - t * 128));
      wrow[2 * t] = wrow[2 * t + 1] = c * ix->d;
    }
  }
  int32_t* dwrow = nullptr;
  if (cudaMalloc(&ix->tile_valid, sizeof(int32_t) * nt) != cudaSuccess) return fail(LV_ENOMEM, "tile_valid");
  LV_CUDA(cudaMallocAsync(&dwrow, sizeof(int32_t) * nt * 3, s));
  LV_CUDA(cudaMemcpyAsync(ix->tile_valid, tv.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(dwrow, wrow.data(), sizeof(int32_t) * nt * 2, cudaMemcpyHostToDevice, s));
  // K6 tile order (C > 1): by the tile's first original row, so the CTAs in flight together read one
  // contiguous window of X (all clusters' rows of it) instead of every C-th row of a wide span
  int32_t* dorder = nullptr;
  if (C > 1) {
    std::vector<int32_t> first(nt), order(nt);
    LV_CUDA(cudaMemcpy2DAsync(first.data(), sizeof(int32_t), ix->perm, 128 * sizeof(int32_t), sizeof(int32_t), nt,
                              cudaMemcpyDeviceToHost, s));
    LV_CUDA(cudaStreamSynchronize(s));
    for (int64_t t = 0; t < nt; ++t) order[t] = (int32_t)t;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return (uint32_t)first[a] < (uint32_t)first[b];   // an all-padding tile (-1) goes last
    });
    dorder = dwrow + 2 * nt;
    LV_CUDA(cudaMemcpyAsync(dorder, order.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
    LV_CUDA(cudaStreamSynchronize(s));   // `order` is pageable and leaves scope
  }
  // X_low = RNE(B_c x) (K6); int8: the fp32 products first, then per-(cluster, coordinate) scales and codes
  const size_t esz = ix->esz();
  if (cudaMalloc(&ix->X_low, esz * ix->n_pad * ix->d) != cudaSuccess) return fail(LV_ENOMEM, "X_low");
  float* xf = nullptr;
  uint32_t* amax = nullptr;
  if (ix->low == LV_I8 && (cudaMalloc(&xf, sizeof(float) * ix->n_pad * ix->d) != cudaSuccess ||
                           cudaMalloc(&amax, sizeof(uint32_t) * (size_t)C * ix->d) != cudaSuccess)) {
    cudaFree(xf);
    return fail(LV_ENOMEM, "lv_encode_database: int8 staging");
  }
  // full-precision copy for the re-rank (allocated before the timed kernels: a host-side
  // cudaMalloc between two event records would count as kernel time)
  const size_t fsz = ix->full == LV_F16 ? 2 : 4;
  if (cudaMalloc(&ix->X_full, fsz * n * ix->D) != cudaSuccess) return fail(LV_ENOMEM, "X_full");
  // fp16 rows: B as row-scaled fp16 planes (built once per operand set, outside the timed window)
  const bool direct = x_dtype == LV_F16 && env_double("LV_K6_DIRECT", 1.0) != 0.0;
  if (direct && !ix->Bh_planes) {
    const int Nc = ix->C * ix->d;
    if (cudaMalloc(&ix->Bh_planes, (size_t)3 * Nc * ix->Kp * 2) != cudaSuccess ||
        cudaMalloc(&ix->b_scale, sizeof(float) * Nc) != cudaSuccess)
      return fail(LV_ENOMEM, "lv_encode_database: fp16 B planes");
    LV_CUDA(lv::launch_split_h(ix->B, Nc, ix->D, ix->Kp, ix->Bh_planes, ix->b_scale, s));
    lv_status hs = make_tmap(&ix->tmap_bh, ix->Bh_planes, 3 * (int64_t)Nc, ix->Kp, lv::encode_kblock(), false, ix->d);
    if (hs) return hs;
  }
  const double hplanes = env_double("LV_K6_HPLANES", 0.0);   // 0: two for bf16 storage, else three
  LV_CUDA(cudaEventRecord(ev[1], s));
  if (direct) {
    const int ot = ix->low == LV_I8 ? 2 : (ix->low == LV_BF16 ? 0 : 1);
    LV_CUDA(lv::launch_encode_h(&ix->tmap_bh, ix->b_scale, X, ix->D, ix->Kp, ix->d, ix->C * ix->d, ix->perm, dwrow, dorder,
                                nt, ix->low == LV_I8 ? (void*)xf : ix->X_low, ot, hplanes >= 3.0, s, n));
    if (ix->low == LV_I8) {
      LV_CUDA(lv::launch_i8_db_scales(xf, nt, ix->d, dwrow, C, amax, ix->i8_delta, s));
      LV_CUDA(lv::launch_i8_db_codes(xf, nt, ix->d, dwrow, ix->i8_delta, reinterpret_cast<int8_t*>(ix->X_low), s));
    }
  } else if (ix->low == LV_I8) {   // (ev[0] is unused: the sort is timed by ev[4..7])
    LV_CUDA(lv::launch_encode_tc(&ix->tmap_b, X, x_dtype == LV_F16, ix->D, ix->Kp, ix->d, ix->C * ix->d, ix->perm, dwrow,
                                 dorder, nt, xf, 2, true, s, n));
    LV_CUDA(lv::launch_i8_db_scales(xf, nt, ix->d, dwrow, C, amax, ix->i8_delta, s));
    LV_CUDA(lv::launch_i8_db_codes(xf, nt, ix->d, dwrow, ix->i8_delta, reinterpret_cast<int8_t*>(ix->X_low), s));
  } else {
    LV_CUDA(lv::launch_encode_tc(&ix->tmap_b, X, x_dtype == LV_F16, ix->D, ix->Kp, ix->d, ix->C * ix->d, ix->perm, dwrow,
                                 dorder, nt, ix->X_low, ix->low == LV_BF16 ? 0 : 1,
                                 env_double("LV_K6_PLANES", 3.0) >= 3.0, s, n));
  }
  LV_CUDA(cudaEventRecord(ev[2], s));
  LV_CUDA(lv::launch_convert(X, x_dtype == LV_F16, ix->X_full, ix->full == LV_F16, n * ix->D, s));
  LV_CUDA(cudaEventRecord(ev[3], s));
  lv_status ts = make_xlow_tmap(ix);
  LV_CUDA(cudaStreamSynchronize(s));
  cudaFree(dwrow);
  cudaFree(xf);
  cudaFree(amax);
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, ev[4], ev[5]);
  cudaEventElapsedTime(&b, ev[6], ev[7]);
  ix->enc_ms[0] = a + b;
  for (int i = 1; i < 3; ++i) cudaEventElapsedTime(&ix->enc_ms[i], ev[i], ev[i + 1]);
  ix->enc_timed = true;
  return ts;
}

lv_status lv_project_queries(const lv_index* ix, const float* Q, int64_t m, void* Qp, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!ix || !Q || !Qp || m <= 0) return fail(LV_EINVAL, "lv_project_queries: bad arguments");
  if (ix->low == LV_I8) return fail(LV_EINVAL, "lv_project_queries: an int8 index needs lv_project_queries_i8");
  if (m > (1 << 24)) return fail(LV_EINVAL, "lv_project_queries: m too large");
  cudaStream_t s = (cudaStream_t)stream;
  const int Cd = ix->C * ix->ds;   // search width (C = 1 when ds < d: the first ds rows of A)
  const int64_t m_pad = (m + 127) / 128 * 128;
  void* planes = nullptr;
  LV_CUDA(cudaMallocAsync(&planes, (size_t)3 * m_pad * ix->Kp * 2, s));
  CUtensorMap tq;
  st = make_tmap(&tq, planes, 3 * m_pad, ix->Kp, 64, true, 128);
  if (st) {
    cudaFreeAsync(planes, s);
    return st;
  }
  LV_CUDA(lv::launch_split3(Q, false, m, m_pad, ix->D, ix->Kp, planes, s));
  LV_CUDA(lv::launch_proj_tc(&tq, &ix->tmap_a, (int)m_pad, Cd, ix->a_rows, ix->Kp, Qp, Cd, (int)m,
                             ix->low == LV_BF16 ? 0 : 1, s));
  LV_CUDA(cudaFreeAsync(planes, s));
  return LV_OK;
}

lv_status lv_project_queries_i8(const lv_index* ix, const float* Q, int64_t m, int8_t* codes, float* scales,
                                void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!ix || !Q || !codes || !scales || m <= 0) return fail(LV_EINVAL, "lv_project_queries_i8: bad arguments");
  if (ix->low != LV_I8) return fail(LV_EINVAL, "lv_project_queries_i8: not an int8 index");
  if (m > (1 << 24)) return fail(LV_EINVAL, "lv_project_queries_i8: m too large");
  cudaStream_t s = (cudaStream_t)stream;
  const int Cd = ix->C * ix->ds;
  const int64_t m_pad = (m + 127) / 128 * 128;
  void* planes = nullptr;
  float* qf = nullptr;
  LV_CUDA(cudaMallocAsync(&planes, (size_t)3 * m_pad * ix->Kp * 2, s));
  LV_CUDA(cudaMallocAsync(&qf, sizeof(float) * (size_t)m_pad * Cd, s));
  CUtensorMap tq;
  st = make_tmap(&tq, planes, 3 * m_pad, ix->Kp, 64, true, 128);
  cudaError_t e = st ? cudaSuccess : lv::launch_split3(Q, false, m, m_pad, ix->D, ix->Kp, planes, s);
  if (!st && e == cudaSuccess)
    e = lv::launch_proj_tc(&tq, &ix->tmap_a, (int)m_pad, Cd, ix->a_rows, ix->Kp, qf, Cd, (int)m, 2, s);
  if (!st && e == cudaSuccess) e = lv::launch_i8_queries(qf, m, ix->C, ix->ds, ix->i8_delta, ix->d, codes, scales, s);
  cudaFreeAsync(planes, s);
  cudaFreeAsync(qf, s);
  if (!st && e != cudaSuccess) st = fail(LV_ECUDA, "lv_project_queries_i8: %s", cudaGetErrorString(e));
  return st;
}

lv_status lv_index_i8_scales(const lv_index* ix, float* delta) {
  if (!ix || !delta) return fail(LV_EINVAL, "lv_index_i8_scales: bad arguments");
  if (ix->low != LV_I8 || ix->n <= 0) return fail(LV_EINVAL, "lv_index_i8_scales: not an encoded int8 index");
  LV_CUDA(cudaMemcpy(delta, ix->i8_delta, sizeof(float) * (size_t)ix->C * ix->d, cudaMemcpyDeviceToHost));
  return LV_OK;
}

// Query batches of at most LV_MAX_BATCH (default 32768) queries bound the search workspace
// (candidate lists ~ 64 x Cap x 8 bytes per query).
static int64_t max_batch() {
  const int64_t v = (int64_t)env_double("LV_MAX_BATCH", 32768.0);
  return std::max<int64_t>(128, v / 128 * 128);
}

static lv_status check_search_args(const lv_index* ix, int64_t m, int32_t k, int32_t R) {
  if (!ix || m <= 0) return fail(LV_EINVAL, "lv_search: bad arguments");
  if (ix->n <= 0) return fail(LV_EINVAL, "lv_search: index not encoded");
  if (k < 1 || k > R || R > 256 || R > ix->n) return fail(LV_EINVAL, "lv_search: need 1 <= k <= R <= min(n, 256)");
  if (m > (1 << 24)) return fail(LV_EINVAL, "lv_search: m too large");
  return LV_OK;
}

// Batch b covers query rows [off_b, off_b + mb): off_b = b * mb, except the last batch, which ends
// at m (it may overlap the previous one; overlapping rows are recomputed with identical results,
// so every batch has the same shape and reuses one plan).
static void batch_layout(int64_t m, int64_t maxB, int64_t* nb, int64_t* mb) {
  if (m <= maxB) {
    *nb = 1;
    *mb = m;
    return;
  }
  int64_t n = (m + maxB - 1) / maxB;
  const int64_t b = ((m + n - 1) / n + 127) / 128 * 128;
  *mb = std::min(b, m);
  *nb = (m + *mb - 1) / *mb;
}

// One search over m <= the batch limit (lv_search splits larger batches).
static lv_status search_batch(lv_index* ix, const float* Q, int64_t m, int32_t k, int32_t R, int32_t* ids,
                              float* scores, lv_search_debug* dbg, void* stream) {
  int nsm = 0;
  lv_status st = check_device(&nsm);
  if (st) return st;
  if (!Q || !ids || !scores) return fail(LV_EINVAL, "lv_search: bad arguments");
  if ((st = check_search_args(ix, m, k, R))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int Cd = ix->C * ix->ds;   // search width (lv_index_set_search_dim)
  PlanCache& pc = ix->plan;
  if (!(pc.valid && pc.m == m && pc.R == R && pc.nsm == nsm)) {
    // new search shape: plan the scan, (re)size the workspace, upload the chunk tables once
    pc.valid = false;
    Plan pl;
    st = plan_search(ix, m, R, nsm, &pl);
    if (st) return st;
    size_t nchunk_ints = pl.repair_chunks.size() + 1;
    for (auto& ch : pl.chunks) nchunk_ints += ch.size() + 1;
    const int NS2 = 4 * pl.NS;   // sub-lists per query
    const size_t mp = pl.m_pad;
    size_t need = (mp * Cd * 2 + 256) + ((size_t)3 * mp * ix->Kp * 2 + 256) + ((size_t)NS2 * mp * pl.Cap * 8 + 256) +
                  ((size_t)NS2 * mp * 4 + 256) +
                  ((size_t)NS2 * mp * 8 + 256) + (mp * 8 + 256) + ((size_t)pl.QP * 16 + 256) + (16 * 4 + 256) + (kMaxScans * 4 + 256) +
                  (mp * (size_t)R * 4 + 256) + (mp * 4 + 256) +
                  (nchunk_ints * 4 + 256 * (pl.chunks.size() + 2));
    if (pl.sampled)
      need += (mp * Cd * 2 + 256) + (mp * 8 + 256) + ((size_t)pl.nblk * mp * 4 + 256) + (2 * mp * 4 + 256);
    if (ix->flex) need += mp * (size_t)ix->D * 4 + 256;
    if (ix->low == LV_I8) need += (mp * (size_t)Cd * 4 + 256) + 2 * (mp * (size_t)ix->C * 4 + 256);
    if (need > ix->ws_bytes) {
      LV_CUDA(cudaStreamSynchronize(s));   // the old workspace may still be in use on s
      cudaFree(ix->ws);
      ix->ws = nullptr;
      ix->ws_bytes = 0;
      if (cudaMalloc(&ix->ws, need) != cudaSuccess) return fail(LV_ENOMEM, "lv_search: workspace %zu bytes", need);
      ix->ws_bytes = need;
    }
    uint8_t* p = reinterpret_cast<uint8_t*>(ix->ws);
    pc.Qp = carve<uint16_t>(p, mp * Cd);
    pc.Qplanes = carve<uint16_t>(p, (size_t)3 * mp * ix->Kp);
    st = make_tmap(&pc.tmap_q, pc.Qplanes, 3 * (int64_t)mp, ix->Kp, 64, true, 128);
    if (st) return st;
    pc.cand = carve<uint64_t>(p, (size_t)NS2 * mp * pl.Cap);
    pc.zero_lo = p;
    pc.cnt = carve<int32_t>(p, (size_t)NS2 * mp);
    pc.tau = carve<uint64_t>(p, (size_t)NS2 * mp);
    pc.tbest = carve<unsigned long long>(p, mp);
    pc.slot_busy = carve<int32_t>(p, (size_t)pl.QP * 4);   // [QP][2] 64-bit sub-list masks (one per query half)
    pc.sel_ids = carve<int32_t>(p, mp * (size_t)R);
    pc.sel_n = carve<int32_t>(p, mp);
    pc.fail = carve<int32_t>(p, 16);
    pc.unit_ctr = carve<int32_t>(p, kMaxScans);
    pc.zero_hi = p;
    if (pl.sampled) {
      pc.Qr = carve<uint16_t>(p, mp * Cd);
      pc.tau2 = carve<uint64_t>(p, mp);
      pc.bmax = carve<float>(p, (size_t)pl.nblk * mp);
      pc.fail_list = carve<int32_t>(p, 2 * mp);
    }
    pc.Qx = ix->flex ? carve<float>(p, mp * (size_t)ix->D) : nullptr;
    pc.Qf = ix->low == LV_I8 ? carve<float>(p, mp * (size_t)Cd) : nullptr;
    pc.qscale = ix->low == LV_I8 ? carve<float>(p, mp * (size_t)ix->C) : nullptr;
    pc.qscale_r = ix->low == LV_I8 ? carve<float>(p, mp * (size_t)ix->C) : nullptr;
    pc.chunk_info.assign(pl.chunks.size(), nullptr);
    for (size_t k = 0; k < pl.chunks.size(); ++k) pc.chunk_info[k] = carve<int32_t>(p, pl.chunks[k].size() + 1);
    pc.repair_info = carve<int32_t>(p, pl.repair_chunks.size() + 1);
    for (size_t k = 0; k < pl.chunks.size(); ++k)
      LV_CUDA(cudaMemcpyAsync(pc.chunk_info[k], pl.chunks[k].data(), pl.chunks[k].size() * 4, cudaMemcpyHostToDevice, s));
    if (!pl.repair_chunks.empty())
      LV_CUDA(cudaMemcpyAsync(pc.repair_info, pl.repair_chunks.data(), pl.repair_chunks.size() * 4,
                              cudaMemcpyHostToDevice, s));
    LV_CUDA(cudaStreamSynchronize(s));   // host vectors are the copy sources
    pc.pl = std::move(pl);
    pc.m = m;
    pc.R = R;
    pc.nsm = nsm;
    pc.valid = true;
  }
  const Plan& pl = pc.pl;
  const int NS2 = 4 * pl.NS;
  void* Qp = pc.Qp;
  const std::vector<int32_t*>& chunk_info = pc.chunk_info;

  // phase marks: 0 start, 1 after K1, 2 after the sample stage, 3 after the threshold select,
  // 4 after the main scan, 5 after K4, 6 after K5, 7 end (after the repairs)
  const int timing = dbg ? dbg->timing : 0;
  std::vector<cudaEvent_t> ev;
  if (timing) {
    for (int i = 0; i < 8; ++i) {
      if (ix->ev_pool.empty()) {
        cudaEvent_t e;
        LV_CUDA(cudaEventCreate(&e));
        ix->ev_pool.push_back(e);
      }
      ev.push_back(ix->ev_pool.back());
      ix->ev_pool.pop_back();
    }
  }
  auto mark = [&](int i) -> lv_status {
    if (timing) LV_CUDA(cudaEventRecord(ev[i], s));
    return LV_OK;
  };
  if ((st = mark(0))) return st;
  int launches = 0;
  LV_CUDA(cudaMemsetAsync(pc.zero_lo, 0, pc.zero_hi - pc.zero_lo, s));
  // K1 projection (rows >= m are zero)
  LV_CUDA(lv::launch_split3(Q, false, m, pl.m_pad, ix->D, ix->Kp, pc.Qplanes, s));
  if (ix->low == LV_I8) {
    // int8 (NEXT-4): q' in fp32, then per (query, view) codes and scales
    LV_CUDA(lv::launch_proj_tc(&pc.tmap_q, &ix->tmap_a, pl.m_pad, Cd, ix->a_rows, ix->Kp, pc.Qf, Cd, pl.m_pad, 2, s));
    LV_CUDA(lv::launch_i8_queries(pc.Qf, pl.m_pad, ix->C, ix->ds, ix->i8_delta, ix->d, reinterpret_cast<int8_t*>(Qp),
                                  pc.qscale, s));
    launches += 3;
  } else {
    LV_CUDA(lv::launch_proj_tc(&pc.tmap_q, &ix->tmap_a, pl.m_pad, Cd, ix->a_rows, ix->Kp, Qp, Cd, pl.m_pad,
                               ix->low == LV_BF16 ? 0 : 1, s));
    launches += 2;
  }
  if (ix->flex) {
    // the re-rank's query side A'q (all D rows of A', fp32): <A'q, x'> = <q, x> (Eq.(12))
    LV_CUDA(lv::launch_proj_tc(&pc.tmap_q, &ix->tmap_a, pl.m_pad, ix->D, ix->a_rows, ix->Kp, pc.Qx, ix->D, pl.m_pad, 2, s));
    ++launches;
  }
  if ((st = mark(1))) return st;
  lv::ScoreArgs sa;
  sa.Qp = Qp;
  sa.C = ix->C;
  sa.m = (int)m;
  sa.m_pad = pl.m_pad;
  sa.QP = pl.QP;
  sa.d = ix->ds;
  sa.R = R;
  sa.NS = NS2;   // the scan claims single sub-lists (64-bit masks per query tile and half)
  sa.Cap = pl.Cap;
  sa.stages = pl.stages;
  sa.tile_valid = ix->tile_valid;
  sa.perm = (ix->C > 1 || ix->flex) ? ix->perm : nullptr;   // keys carry original / external ids
  sa.qscale = pc.qscale;
  sa.cand = pc.cand;
  sa.cnt = pc.cnt;
  sa.tau = pc.tau;
  sa.tbest = pc.tbest;
  sa.raw = dbg ? dbg->raw_scores : nullptr;
  sa.bmax = nullptr;
  sa.m_dev = nullptr;
  sa.n_pad = ix->n_pad;
  sa.slot_busy = pc.slot_busy;
  {
    const char* f = getenv("LV_DEBUG_SCAN_FLAGS");
    sa.flags = f ? atoi(f) : 0;
  }
  unsigned long long*& dstats = ix->dbg_stats;   // debug counters (LV_DEBUG_SCAN_FLAGS & 2), owned by the index
  sa.stats = nullptr;
  if (sa.flags & (2 | 128)) {
    if (!dstats) LV_CUDA(cudaMalloc(&dstats, 16 * sizeof(unsigned long long)));
    sa.stats = dstats;
  }
  int nscan = 0;
  const bool dyn_units = env_double("LV_DYN_UNITS", 1.0) != 0.0;
  auto scan = [&](const int32_t* info, const std::vector<int32_t>& host_chunks, int qtiles, const char* what) -> lv_status {
    sa.P = (int)(host_chunks.size() / lv::kChunkInts);
    sa.chunk_info = info;
    const int grid = (int)std::min<int64_t>(nsm, (int64_t)sa.P * qtiles);
    if (grid <= 0) return LV_OK;
    // dynamic unit order (LV_DYN_UNITS, default on): a fresh zeroed counter per launch
    sa.unit_ctr = (dyn_units && nscan < kMaxScans) ? pc.unit_ctr + nscan : nullptr;
    ++nscan;
    if (sa.stats) LV_CUDA(cudaMemsetAsync(sa.stats, 0, 16 * sizeof(unsigned long long), s));
    LV_CUDA(lv::launch_score(&ix->tmap_xlow_s, sa, ix->fmt(), grid, pl.smem, s));
    ++launches;
    if (sa.stats) {
      unsigned long long h[16];
      LV_CUDA(cudaMemcpyAsync(h, sa.stats, sizeof h, cudaMemcpyDeviceToHost, s));
      LV_CUDA(cudaStreamSynchronize(s));
      int64_t tiles = 0;
      for (int c = 0; c < sa.P; ++c) {
        const int32_t* ci = host_chunks.data() + lv::kChunkInts * c;
        tiles += (ci[1] - ci[0] + ci[3] - 1) / ci[3];
      }
      if (sa.flags & 128)
        fprintf(stderr,
                "[lv] %s: P=%d tiles=%lld grid=%d per MMA-tile cycles: wait acc_empty+b_full %.1f, issue->next %.1f "
                "(tiles %llu); per epilogue job: wait acc_full %.1f, total %.1f (jobs %llu); append entries %llu "
                "(%.3f per job) of %.1f cycles each\n",
                what, sa.P, (long long)tiles, grid, (double)h[0] / h[5], (double)h[4] / h[5], h[5],
                (double)h[2] / h[6], (double)h[7] / h[6], h[6], h[1], (double)h[1] / h[6], (double)h[3] / (h[1] ? h[1] : 1));
      if (sa.flags & 128)
        fprintf(stderr,
                "[lv] %s: append batches %llu, per batch: read %.1f, process %.1f cycles; pushes %llu of %.1f cycles "
                "(room waits %.1f)\n",
                what, h[8], (double)h[9] / (h[8] ? h[8] : 1), (double)h[10] / (h[8] ? h[8] : 1), h[11],
                (double)h[12] / (h[11] ? h[11] : 1), (double)h[13] / (h[11] ? h[11] : 1));
      else
        fprintf(stderr, "[lv] %s: P=%d tiles=%lld grid=%d hit_warp_tiles=%llu appends=%llu compactions=%llu wait_spins=%llu\n",
                what, sa.P, (long long)tiles, grid, h[0], h[1], h[2], h[3]);
    }
    return LV_OK;
  };
  lv::RerankArgs ra;
  ra.m = (int)m;
  ra.m_pad = pl.m_pad;
  ra.D = ix->D;
  ra.R = R;
  ra.k = k;
  ra.NS = NS2;
  ra.Cap = pl.Cap;
  ra.cand = pc.cand;
  ra.cnt = pc.cnt;
  ra.Q = ix->flex ? pc.Qx : Q;                 // flex: <A'q, x'> (Eq.(12)); else <q, x>
  ra.X = ix->X_full;
  ra.full_f16 = ix->full == LV_F16;
  ra.row_of_id = ix->flex ? ix->inv : nullptr;
  ra.ids = ids;
  ra.scores = scores;
  ra.cand_ids = dbg ? dbg->cand_ids : nullptr;
  ra.cand_scores = dbg ? dbg->cand_scores : nullptr;
  ra.qmap = nullptr;
  ra.m_dev = nullptr;
  ra.checked = 0;
  ra.fail_count = nullptr;
  ra.fail_list = nullptr;
  ra.sel_ids = pc.sel_ids;
  ra.sel_n = pc.sel_n;
  if (!pl.sampled) {
    // staged path: geometric stages with exact threshold merges in between
    if ((st = mark(2)) || (st = mark(3))) return st;
    for (size_t k = 0; k < pl.chunks.size(); ++k) {
      char nm[32];
      snprintf(nm, sizeof nm, "stage %zu", k);
      st = scan(chunk_info[k], pl.chunks[k], pl.QP, nm);
      if (st) return st;
      if (k + 1 < pl.chunks.size()) {
        LV_CUDA(lv::launch_tau_merge(pc.cand, pc.cnt, pc.tau, NS2, (int)m, pl.m_pad, pl.Cap, R, s));
        ++launches;
      }
    }
    if ((st = mark(4))) return st;
    LV_CUDA(lv::launch_select_topr(ra, s));
    if ((st = mark(5))) return st;
    LV_CUDA(lv::launch_rerank_topk(ra, s));
    if ((st = mark(6))) return st;
    launches += 2;
  } else {
    // sampled path: (1) sample stage -> block maxima; (2) per-query threshold with >= j1 rows
    // above it; (3) one main stage with that threshold; (4) exactness check in the re-rank;
    // (5) repair of the failed queries with the looser j2 threshold, then with none
    sa.bmax = pc.bmax;
    const int flags0 = sa.flags;
    if (pl.fine_blocks) sa.flags |= 8;
    st = scan(chunk_info[0], pl.chunks[0], pl.QP, "sample");
    if (st) return st;
    sa.flags = flags0;
    sa.bmax = nullptr;
    if ((st = mark(2))) return st;
    LV_CUDA(lv::launch_bmax_select(pc.bmax, pl.nblk, (int)m, pl.m_pad, pl.j1, pl.j2, pc.tau, pc.cnt, NS2, pc.tau2, s));
    ++launches;
    if ((st = mark(3))) return st;
    st = scan(chunk_info[1], pl.chunks[1], pl.QP, "main");
    if (st) return st;
    if ((st = mark(4))) return st;
    ra.checked = 1;
    ra.fail_count = pc.fail + 0;
    ra.fail_list = pc.fail_list;
    LV_CUDA(lv::launch_select_topr(ra, s));
    if ((st = mark(5))) return st;
    LV_CUDA(lv::launch_rerank_topk(ra, s));
    if ((st = mark(6))) return st;
    launches += 2;
    for (int round = 0; round < 2; ++round) {
      int32_t* flist = pc.fail_list + (size_t)round * pl.m_pad;
      int32_t* fcount = pc.fail + round;
      int32_t* mdev = pc.fail + 4 + round;
      LV_CUDA(lv::launch_repair_setup(Qp, Cd * ix->esz() / 2, flist, fcount, pc.Qr, round == 0 ? pc.tau2 : nullptr,
                                      pc.tau, pc.tbest, pc.cnt, NS2, pl.m_pad, (int)m, mdev, pc.qscale, pc.qscale_r, ix->C, s));
      sa.Qp = pc.Qr;
      sa.qscale = pc.qscale_r;
      sa.m_dev = mdev;
      st = scan(pc.repair_info, pl.repair_chunks, 1, round == 0 ? "repair-1" : "repair-2");
      if (st) return st;
      ra.qmap = flist;
      ra.m_dev = mdev;
      ra.checked = round == 0 ? 1 : 0;
      ra.fail_count = pc.fail + 1;
      ra.fail_list = pc.fail_list + pl.m_pad;
      LV_CUDA(lv::launch_select_topr(ra, s));
      LV_CUDA(lv::launch_rerank_topk(ra, s));
      launches += 3;
    }
    sa.Qp = Qp;
    sa.qscale = pc.qscale;
    sa.m_dev = nullptr;
    if (sa.stats) {
      int32_t hf[2];
      LV_CUDA(cudaMemcpyAsync(hf, pc.fail, sizeof hf, cudaMemcpyDeviceToHost, s));
      LV_CUDA(cudaStreamSynchronize(s));
      fprintf(stderr, "[lv] sampled: stride=%d nblk=%d j1=%d j2=%d failed=%d then %d\n", pl.stride, pl.nblk, pl.j1,
              pl.j2, hf[0], hf[1]);
    }
  }
  if ((st = mark(7))) return st;
  if (timing == 1) {
    LV_CUDA(cudaEventSynchronize(ev[7]));
    float t[7];
    for (int i = 0; i < 7; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    for (int i = 0; i < 7; ++i) dbg->kernel_ms[i] = t[i];
    cudaEventElapsedTime(&dbg->kernel_ms[7], ev[0], ev[7]);
    dbg->phase_ms[0] = t[0];
    dbg->phase_ms[1] = t[1] + t[2] + t[3];
    dbg->phase_ms[2] = t[4] + t[5] + t[6];
    dbg->phase_ms[3] = dbg->kernel_ms[7];
    for (auto e : ev) ix->ev_pool.push_back(e);
  } else if (timing == 2) {
    ix->ev_pending.push_back(ev);
  }
  if (dbg) {
    dbg->path = pl.sampled ? 1 : 0;
    dbg->failed[0] = dbg->failed[1] = 0;
    if (timing && pl.sampled) {
      int32_t hf[2];
      LV_CUDA(cudaMemcpyAsync(hf, pc.fail, sizeof hf, cudaMemcpyDeviceToHost, s));
      LV_CUDA(cudaStreamSynchronize(s));
      dbg->failed[0] = hf[0];
      dbg->failed[1] = hf[1];
    }
    dbg->launches = launches;
    dbg->slots = NS2;
    dbg->units = pl.total_units;
    dbg->grid = pl.grid;
  }
  return LV_OK;
}

lv_status lv_encode_timing(const lv_index* ix, float* ms) {
  if (!ix || !ms) return fail(LV_EINVAL, "lv_encode_timing: bad arguments");
  if (!ix->enc_timed) return fail(LV_EINVAL, "lv_encode_timing: no encode has run");
  for (int i = 0; i < 3; ++i) ms[i] = ix->enc_ms[i];
  return LV_OK;
}

lv_status lv_timing_collect(lv_index* ix, float* kernel_ms, int32_t* calls) {
  if (!ix || !kernel_ms) return fail(LV_EINVAL, "lv_timing_collect: bad arguments");
  double acc[8] = {0};
  const int n = (int)ix->ev_pending.size();
  for (auto& g : ix->ev_pending) {
    LV_CUDA(cudaEventSynchronize(g[7]));
    float t;
    for (int i = 0; i < 7; ++i) {
      cudaEventElapsedTime(&t, g[i], g[i + 1]);
      acc[i] += t;
    }
    cudaEventElapsedTime(&t, g[0], g[7]);
    acc[7] += t;
    for (auto e : g) ix->ev_pool.push_back(e);
  }
  ix->ev_pending.clear();
  for (int i = 0; i < 8; ++i) kernel_ms[i] = n ? (float)(acc[i] / n) : 0.f;
  if (calls) *calls = n;
  return LV_OK;
}

lv_status lv_search(lv_index* ix, const float* Q, int64_t m, int32_t k, int32_t R, int32_t* ids, float* scores,
                    lv_search_debug* dbg, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!Q || !ids || !scores) return fail(LV_EINVAL, "lv_search: bad arguments");
  if ((st = check_search_args(ix, m, k, R))) return st;
  int64_t nb, mb;
  batch_layout(m, max_batch(), &nb, &mb);
  if (nb == 1) return search_batch(ix, Q, m, k, R, ids, scores, dbg, stream);
  if (dbg && dbg->raw_scores) return fail(LV_EINVAL, "lv_search: raw_scores needs m <= LV_MAX_BATCH");
  lv_search_debug acc{};
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t off = (b + 1 < nb) ? b * mb : m - mb;
    lv_search_debug db{};
    if (dbg) {
      db = *dbg;
      if (dbg->cand_ids) db.cand_ids = dbg->cand_ids + off * R;
      if (dbg->cand_scores) db.cand_scores = dbg->cand_scores + off * R;
    }
    st = search_batch(ix, Q + off * ix->D, mb, k, R, ids + off * k, scores + off * k, dbg ? &db : nullptr, stream);
    if (st) return st;
    if (dbg) {
      for (int i = 0; i < 4; ++i) acc.phase_ms[i] += db.phase_ms[i];
      for (int i = 0; i < 8; ++i) acc.kernel_ms[i] += db.kernel_ms[i];
      acc.failed[0] += db.failed[0];
      acc.failed[1] += db.failed[1];
      acc.launches += db.launches;
      acc.units += db.units;
      acc.slots = db.slots;
      acc.grid = db.grid;
      acc.path = db.path;
    }
  }
  if (dbg) {
    for (int i = 0; i < 4; ++i) dbg->phase_ms[i] = acc.phase_ms[i];
    for (int i = 0; i < 8; ++i) dbg->kernel_ms[i] = acc.kernel_ms[i];
    dbg->failed[0] = acc.failed[0];
    dbg->failed[1] = acc.failed[1];
    dbg->launches = acc.launches;
    dbg->units = acc.units;
    dbg->slots = acc.slots;
    dbg->grid = acc.grid;
    dbg->path = acc.path;
  }
  return LV_OK;
}

lv_status lv_search_host(lv_index* ix, const float* Q_host, int64_t m, int32_t k, int32_t R, int32_t* ids_host,
                         float* scores_host, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!Q_host || !ids_host || !scores_host) return fail(LV_EINVAL, "lv_search_host: bad arguments");
  if ((st = check_search_args(ix, m, k, R))) return st;   // before any copy is enqueued
  cudaStream_t s = (cudaStream_t)stream;
  const size_t qb = (size_t)m * ix->D * 4, ob = (size_t)m * k * 4;
  const size_t need = qb + 2 * ob + 1024;
  if (need > ix->hs_bytes) {
    LV_CUDA(cudaStreamSynchronize(s));
    cudaFree(ix->hs);
    ix->hs = nullptr;
    ix->hs_bytes = 0;
    if (cudaMalloc(&ix->hs, need) != cudaSuccess) return fail(LV_ENOMEM, "lv_search_host: staging");
    ix->hs_bytes = need;
  }
  if (!ix->cs) {
    LV_CUDA(cudaStreamCreateWithFlags(&ix->cs, cudaStreamNonBlocking));
    for (int i = 0; i < kHostEv; ++i) LV_CUDA(cudaEventCreateWithFlags(&ix->hev[i], cudaEventDisableTiming));
  }
  uint8_t* p = reinterpret_cast<uint8_t*>(ix->hs);
  float* dQ = carve<float>(p, (size_t)m * ix->D);
  int32_t* dI = carve<int32_t>(p, (size_t)m * k);
  float* dS = carve<float>(p, (size_t)m * k);
  // two query batches when the batch is large: batch 1's upload (copy stream) overlaps batch 0's
  // search, batch 0's download overlaps batch 1's search
  int64_t nb = 1, mb = m;
  // LV_HOST_BATCHES: equal query batches (1: one batch, no copy/compute overlap), each >= 2048 queries
  const int64_t nh = std::max<int64_t>(1, std::min<int64_t>(kHostEv - 2, (int64_t)env_double("LV_HOST_BATCHES", 2.0)));
  const int64_t want = std::min<int64_t>(nh, std::max<int64_t>(1, m / 2048));
  if (want >= 2) batch_layout(m, std::min<int64_t>(max_batch(), (m + want - 1) / want + 127), &nb, &mb);
  if (nb > kHostEv - 2) batch_layout(m, max_batch(), &nb, &mb);
  if (nb > kHostEv - 2) return fail(LV_EUNSUPPORTED, "lv_search_host: m=%lld needs more than %d batches", (long long)m, kHostEv - 2);
  const int64_t D = ix->D;
  std::vector<int64_t> lo(nb), hi(nb), off(nb);
  for (int64_t b = 0; b < nb; ++b) {
    off[b] = (b + 1 < nb) ? b * mb : m - mb;
    lo[b] = b == 0 ? 0 : hi[b - 1];   // rows first needed by batch b
    hi[b] = off[b] + mb;
  }
  // events: [b] upload of batch b's rows done (copy stream), [kHostEv - 2] start, [kHostEv - 1]
  // search of the current batch done
  cudaEvent_t* ev = ix->hev;
  cudaEvent_t ev_start = ev[kHostEv - 2], ev_done = ev[kHostEv - 1];
  LV_CUDA(cudaEventRecord(ev_start, s));          // the copy stream starts after prior work on s
  LV_CUDA(cudaStreamWaitEvent(ix->cs, ev_start, 0));
  for (int64_t b = 0; b < nb; ++b) {
    // uploads: batch b's new rows on the copy stream
    LV_CUDA(cudaMemcpyAsync(dQ + lo[b] * D, Q_host + lo[b] * D, (size_t)(hi[b] - lo[b]) * D * 4, cudaMemcpyHostToDevice,
                            ix->cs));
    LV_CUDA(cudaEventRecord(ev[b], ix->cs));
  }
  int64_t done = 0;
  for (int64_t b = 0; b < nb; ++b) {
    LV_CUDA(cudaStreamWaitEvent(s, ev[b], 0));
    st = search_batch(ix, dQ + off[b] * D, mb, k, R, dI + off[b] * k, dS + off[b] * k, nullptr, stream);
    if (st) {
      cudaStreamSynchronize(ix->cs);
      return st;
    }
    // downloads of the rows no later batch rewrites: [done, off[b + 1]) (the last batch: to m)
    const int64_t r1 = (b + 1 < nb) ? off[b + 1] : m;
    LV_CUDA(cudaEventRecord(ev_done, s));
    LV_CUDA(cudaStreamWaitEvent(ix->cs, ev_done, 0));
    if (r1 > done) {
      LV_CUDA(cudaMemcpyAsync(ids_host + done * k, dI + done * k, (size_t)(r1 - done) * k * 4, cudaMemcpyDeviceToHost,
                              ix->cs));
      LV_CUDA(cudaMemcpyAsync(scores_host + done * k, dS + done * k, (size_t)(r1 - done) * k * 4,
                              cudaMemcpyDeviceToHost, ix->cs));
      done = r1;
    }
  }
  LV_CUDA(cudaStreamSynchronize(ix->cs));
  LV_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

lv_status lv_assign_tags(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, const float* centres, int32_t C,
                         int32_t* assign, void* stream) {
  return lv_kmeans_assign(X, x_dtype, n, D, centres, C, assign, nullptr, 0, stream);
}

lv_status lv_kmeans_assign(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, const float* centres, int32_t C,
                           int32_t* assign, float* best, int32_t accumulate, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!X || !centres || (!assign && !best) || n <= 0 || D <= 0 || C < 1)
    return fail(LV_EINVAL, "lv_kmeans_assign: bad arguments");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_kmeans_assign: x_dtype must be F32/F16");
  LV_CUDA(lv::launch_assign(X, x_dtype == LV_F16, n, D, centres, C, assign, best, accumulate ? 1 : 0,
                            (cudaStream_t)stream));
  return LV_OK;
}

lv_status lv_normalize_rows(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, float* Xn, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!X || !Xn || n <= 0 || D <= 0) return fail(LV_EINVAL, "lv_normalize_rows: bad arguments");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_normalize_rows: x_dtype must be F32/F16");
  LV_CUDA(lv::launch_normalize(X, x_dtype == LV_F16, n, D, Xn, (cudaStream_t)stream));
  return LV_OK;
}

lv_status lv_kmeans_centre_sums(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, const int32_t* assign,
                                int32_t C, double* sums, int64_t* counts, void* stream) {
  lv_status st = check_device();
  if (st) return st;
  if (!X || !assign || !sums || !counts || n <= 0 || D <= 0 || C < 1)
    return fail(LV_EINVAL, "lv_kmeans_centre_sums: bad arguments");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_kmeans_centre_sums: x_dtype must be F32/F16");
  if (lv::centre_sums_smem(C) > 200 * 1024) return fail(LV_EUNSUPPORTED, "lv_kmeans_centre_sums: C=%d > 384", C);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rpc = 2048;   // rows per chunk
  const int nch = (int)((n + rpc - 1) / rpc);
  float* part = nullptr;
  int32_t* pc = nullptr;
  double* dsum = nullptr;
  long long* dcnt = nullptr;
  LV_CUDA(cudaMallocAsync(&part, sizeof(float) * (size_t)nch * C * D, s));
  LV_CUDA(cudaMallocAsync(&pc, sizeof(int32_t) * (size_t)nch * C, s));
  LV_CUDA(cudaMallocAsync(&dsum, sizeof(double) * (size_t)C * D, s));
  LV_CUDA(cudaMallocAsync(&dcnt, sizeof(long long) * (size_t)C, s));
  cudaError_t e = lv::launch_centre_sums(X, x_dtype == LV_F16, n, D, assign, C, rpc, nch, part, pc, dsum, dcnt, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(sums, dsum, sizeof(double) * (size_t)C * D, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(counts, dcnt, sizeof(long long) * (size_t)C, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(part, s);
  cudaFreeAsync(pc, s);
  cudaFreeAsync(dsum, s);
  cudaFreeAsync(dcnt, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(LV_ECUDA, "lv_kmeans_centre_sums: %s", cudaGetErrorString(e));
  return LV_OK;
}

lv_status lv_index_set_search_dim(lv_index* ix, int32_t d_search) {
  if (!ix) return fail(LV_EINVAL, "lv_index_set_search_dim: bad arguments");
  if (d_search <= 0) d_search = ix->d;
  if (d_search > ix->d) return fail(LV_EINVAL, "lv_index_set_search_dim: d_search=%d > stored d=%d", d_search, ix->d);
  if (d_search != ix->d && ix->C != 1)
    return fail(LV_EINVAL, "lv_index_set_search_dim: a prefix search needs C = 1 (LeanVec-Sphering, §3.1)");
  if (d_search % 32 != 0 || d_search > 192)
    return fail(LV_EINVAL, "lv_index_set_search_dim: d_search=%d not in {32, 64, ..., 192}", d_search);
  if (d_search == ix->ds) return LV_OK;
  ix->ds = d_search;
  ix->plan.valid = false;   // the scan plan depends on the width
  return ix->X_low ? make_search_tmap(ix) : LV_OK;
}

lv_status lv_index_get_search_dim(const lv_index* ix, int32_t* d_search) {
  if (!ix || !d_search) return fail(LV_EINVAL, "lv_index_get_search_dim: bad arguments");
  *d_search = ix->ds;
  return LV_OK;
}

lv_status lv_index_info(const lv_index* ix, int64_t* n, int64_t* n_pad, int32_t* D, int32_t* d, int32_t* C) {
  if (!ix) return fail(LV_EINVAL, "lv_index_info: NULL index");
  if (n) *n = ix->n;
  if (n_pad) *n_pad = ix->n_pad;
  if (D) *D = ix->D;
  if (d) *d = ix->d;
  if (C) *C = ix->C;
  return LV_OK;
}

lv_status lv_index_export(const lv_index* ix, void* X_low, int32_t* perm, int64_t* offsets, void* stream) {
  if (!ix) return fail(LV_EINVAL, "lv_index_export: NULL index");
  if (ix->n <= 0) return fail(LV_EINVAL, "lv_index_export: index not encoded");
  cudaStream_t s = (cudaStream_t)stream;
  if (X_low)
    LV_CUDA(cudaMemcpyAsync(X_low, ix->X_low, (size_t)ix->n_pad * ix->d * ix->esz(), cudaMemcpyDeviceToDevice, s));
  if (perm) LV_CUDA(cudaMemcpyAsync(perm, ix->perm, (size_t)ix->n_pad * 4, cudaMemcpyDeviceToDevice, s));
  if (offsets) std::copy(ix->offsets.begin(), ix->offsets.end(), offsets);
  LV_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

lv_status lv_index_export_full(const lv_index* ix, void* X_full, void* stream) {
  if (!ix || !X_full) return fail(LV_EINVAL, "lv_index_export_full: NULL argument");
  if (ix->flex) return fail(LV_EINVAL, "lv_index_export_full: a flexible index stores x' (lv_index_export_xprime)");
  if (ix->n <= 0 || !ix->X_full) return fail(LV_EINVAL, "lv_index_export_full: index not encoded");
  cudaStream_t s = (cudaStream_t)stream;
  LV_CUDA(cudaMemcpyAsync(X_full, ix->X_full, (size_t)ix->n * ix->D * (ix->full == LV_F16 ? 2 : 4),
                          cudaMemcpyDeviceToDevice, s));
  LV_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

void lv_index_destroy(lv_index* ix) {
  if (!ix) return;
  free_db(ix);
  cudaFree(ix->inv);
  cudaFree(ix->KQ);
  cudaFree(ix->KX);
  cudaFree(ix->A);
  cudaFree(ix->B);
  cudaFree(ix->i8_delta);
  cudaFree(ix->dbg_stats);
  cudaFree(ix->A_planes);
  cudaFree(ix->B_planes);
  cudaFree(ix->Bh_planes);
  cudaFree(ix->b_scale);
  for (auto& g : ix->ev_pending)
    for (auto e : g) cudaEventDestroy(e);
  for (auto e : ix->ev_pool) cudaEventDestroy(e);
  cudaFree(ix->ws);
  cudaFree(ix->hs);
  for (auto e : ix->hev)
    if (e) cudaEventDestroy(e);
  if (ix->cs) cudaStreamDestroy(ix->cs);
  delete ix;
}

}  // extern "C"
