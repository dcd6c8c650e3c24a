// vy_tile.cuh — the fused environment transition on a shared-memory tile.
//
// Semantics: voltyard/backends/_kernel.pyx:239-649 (== pykernel.py:30-429).
//
// Mapping.  One thread per environment; a warp owns a tile of 32 consecutive
// envs.  The tile's per-port state (float64 i_drawn/soc/de, int16 dwell time,
// uint8 meta) and its uint8 action rows are staged from HBM into the warp's
// shared-memory tile with 16-byte cp.async copies ([port][field][lane]
// columns, so per-lane accesses are bank-conflict free).  The per-port phases
// run as rolled loops over the runtime port count (one kernel for every
// station size; the hot code is a few KB — a fully unrolled port loop
// overflowed the instruction cache), per-env scalars live in registers.
//
// Exactness.  All continuous arithmetic is float64 in the reference's
// operation order, built with --fmad=false (explicit FMAs appear only inside
// div_rcp, whose result is the correctly rounded quotient); sums the
// reference accumulates sequentially (tree node loads, energy flows,
// satisfaction penalties) are accumulated sequentially here too, in port
// order.  Each env's trajectory is therefore bit-identical to the reference's
// compiled kernel.
#pragma once

#include "vy_device.cuh"




namespace vy {

// Dynamic shared memory of every kernel in this library.  Tile data is
// accessed with explicit 32-bit shared-window addresses (ld/st.shared via
// inline PTX): pointer arithmetic on the extern array made the compiler
// re-materialise the window base (S2R CgaCtaId + LEA) at every predicated
// access.  The asm is volatile so tile accesses keep program order.
extern __shared__ __align__(128) unsigned char vy_smem[];

// shared-window address of vy_smem, produced by opaque asm so it lives in a
// register instead of being re-materialised at every use
__device__ __forceinline__ uint32_t smem_base() {
  uint32_t a;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(vy_smem));
  return a;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }
__device__ __forceinline__ int lds_s16(uint32_t a) {
  int16_t v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_s16(uint32_t a, int v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v));
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v)); }

// The per-CTA car-profile table in shared memory, addressed through an
// explicit 32-bit shared-window address (a generic Profile* made the compiler
// re-derive the window base, S2UR SR_CgaCtaId + LEA, at every lookup).  Loads
// are non-volatile: the table is read-only after staging.
struct Prof {
  uint32_t a;  // shared address of profile 0
  __device__ __forceinline__ double at(int c, int w) const {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a + (uint32_t)c * (uint32_t)sizeof(Profile) + 8u * w));
    return v;
  }
  __device__ __forceinline__ double cap(int c) const { return at(c, 0); }
  __device__ __forceinline__ double r_ac(int c) const { return at(c, 1); }
  __device__ __forceinline__ double r_dc(int c) const { return at(c, 2); }
  __device__ __forceinline__ double tau(int c) const { return at(c, 3); }
  __device__ __forceinline__ double omt(int c) const { return at(c, 4); }
  __device__ __forceinline__ double rcp_cap(int c) const { return at(c, 5); }
  __device__ __forceinline__ double rcp_omt(int c) const { return at(c, 6); }
  __device__ __forceinline__ double cum(int c) const { return at(c, 7); }
};

// Per-port constants staged in shared memory (one 96-byte record per port):
// every lane reads the same address (broadcast), two doubles per 16-byte
// load, instead of one indexed constant-bank load per value.
struct PortC {
  uint32_t a;  // shared address of port 0's record
  __device__ __forceinline__ void pair(int i, int w, double& x, double& y) const {
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + (uint32_t)i * (8u * kPortWords) + 16u * w));
  }
};

// The capacity tree staged in shared memory, one 32-byte record per node in
// the deepest-first order of the rescale (_kernel.pyx:626-649):
// {cap, eta, RN(1/eta), (lo, hi) slot range}.  Read at a uniform address
// (broadcast) instead of register-indexed constant-bank loads.
struct TreeC {
  uint32_t a;
  __device__ __forceinline__ void rec(int q, double& cap, double& eta, double& rcp_eta, int& lo, int& hi) const {
    const uint32_t r = a + (uint32_t)q * 32u;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(cap), "=d"(eta) : "r"(r));
    asm("ld.shared.f64 %0, [%1];" : "=d"(rcp_eta) : "r"(r + 16u));
    asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(r + 24u));
  }
};

// Global loads issued exactly where written (volatile asm): the compiler
// otherwise sinks early loads next to their first use at the end of the step,
// exposing the full DRAM latency there instead of overlapping it with the
// tile copies.  The per-env state scalars are read once per step (.lu, last
// use); the read-only series go through the non-coherent path (.nc).
__device__ __forceinline__ double ldg_f64(const double* p) {
  double v;
  asm volatile("ld.global.lu.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_nc_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_s32(const int32_t* p) {
  int v;
  asm volatile("ld.global.lu.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_nc_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ldg_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.lu.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_nc_s8(const int8_t* p) {
  int v;
  asm volatile("ld.global.nc.s8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// streamed-tile loads (Spec<4>): per-lane coalesced reads of a port's state,
// issued a few ports ahead of their use (volatile: kept where written)
__device__ __forceinline__ double ldg_st_f64(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_st_s16(const int16_t* p) {
  int16_t v;
  asm volatile("ld.global.s16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

struct EnvRegs {
  int step, day;
  uint64_t akey;
  double b_i, b_soc;
  double ep_profit, ep_reward, ep_missing, ep_energy;
  int ep_overtime, ep_declined, ep_departures;
};

// proxies so tile fields read and assign like lvalues
struct SF64 {
  uint32_t a;
  __device__ __forceinline__ operator double() const { return lds_f64(a); }
  __device__ __forceinline__ void operator=(double v) const { sts_f64(a, v); }
};
struct SS16 {
  uint32_t a;
  __device__ __forceinline__ operator int() const { return lds_s16(a); }
  __device__ __forceinline__ void operator=(int v) const { sts_s16(a, v); }
};
struct SU8 {
  uint32_t a;
  __device__ __forceinline__ operator uint32_t() const { return lds_u8(a); }
  __device__ __forceinline__ void operator=(uint32_t v) const { sts_u8(a, v); }
};

// One lane's view of its warp's tile.  Plain C++ references into vy_smem
// (the compiler infers the shared address space and emits LDS/STS) so loads
// of one port may be scheduled ahead of stores to another in unrolled loops.
struct Lane {
  uint32_t t;  // byte offset of the warp's tile in vy_smem
  double* p;   // this lane's i_drawn slot of port 0 (soc at +32, de at +64 doubles; ports 96 apart)
  int16_t* d;  // this lane's dwell entry of port 0 (ports 32 apart)
  uint8_t* m;  // this lane's meta entry of port 0 (ports 32 apart)
  int lane;
  const TileLayout* L;
  int ps;      // doubles between ports' slots (96; 32 in a streamed tile, which holds i_drawn only)
  __device__ __forceinline__ double& idr(int i) const { return p[i * ps]; }
  __device__ __forceinline__ double& soc(int i) const { return p[i * ps + 32]; }
  __device__ __forceinline__ double& de(int i) const { return p[i * ps + 64]; }
  __device__ __forceinline__ int16_t& dtrem(int i) const { return d[i * 32]; }
  __device__ __forceinline__ uint8_t& meta(int i) const { return m[i * 32]; }
};

__device__ __forceinline__ Lane make_lane(const Params& P, uint32_t tile, int lane) {
  unsigned char* b = vy_smem + tile;
  return Lane{tile, reinterpret_cast<double*>(b + P.L.ports + lane * 8),
              reinterpret_cast<int16_t*>(b + P.L.dtrem + lane * 2), b + P.L.meta + lane, lane, &P.L, P.L.ps / 8};
}

// ---- tile stage-in: bulk copies (TMA engine) completing on a per-warp mbarrier ----
//
// Each (field, port) column of a 32-env tile is one contiguous, aligned run
// in the port-major global layout (256 B of float64, 64 B of int16 dwell, 32
// B of meta), and the tile's uint8 action rows are one contiguous block.  A
// lane issues whole columns as cp.async.bulk copies (one instruction per
// column instead of one 16-byte cp.async per lane and chunk, no per-lane
// address math); they complete on the warp's mbarrier with the expected byte
// count armed by lane 0, and the warp waits on the barrier's phase.
__device__ __forceinline__ void mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "VY_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra VY_WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t sdst, const void* gsrc, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sdst),
               "l"(gsrc), "r"(bytes), "r"(bar)
               : "memory");
}
// generic-proxy accesses of this thread to shared memory are ordered before
// later async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// The step kernel's two-stage load keeps 16-byte cp.async copies: issuing the
// same columns as bulk copies measured slower on B200 (2^20 envs, mid-day
// window: +5% step time for the meta stage as bulk copies, +8.5% for the
// port slots — 32-256 byte copies, ~80 per tile; scripts/ab_roll.sh,
// profiles/r2_bulk_ab.txt).  Rollout and reset kernels load their tile once
// with bulk copies.  -DVY_BULK_META=1 / -DVY_BULK_SLOTS=1 select the bulk variants.
#ifndef VY_BULK_META
#define VY_BULK_META 0
#endif
#ifndef VY_BULK_SLOTS
#define VY_BULK_SLOTS 0
#endif
__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// The warp's barrier: shared address and the parity of its next phase.
struct WarpBar {
  uint32_t a;
  uint32_t phase;
  bool armed;  // a stage is in flight (tile_wait waits for it)
};
__device__ __forceinline__ WarpBar warp_bar_init(const Params& P, uint32_t toff, int lane) {
  WarpBar wb{smem_base() + toff + (uint32_t)P.L.bar, 0u, false};
  if (lane == 0) {
    mbar_init(wb.a);
    mbar_init_fence();
  }
  __syncwarp();
  return wb;
}
__device__ __forceinline__ void bar_wait(WarpBar& wb) {
  if (wb.armed) {
    mbar_wait(wb.a, wb.phase);
    wb.phase ^= 1u;
    wb.armed = false;
  }
}

// the n port columns of every field plus the action rows (rollout / reset: one stage)
__device__ __forceinline__ void tile_issue(const Params& P, uint32_t toff, int64_t b0, int lane, bool with_acts,
                                           WarpBar& wb) {
  const uint32_t t = smem_base() + toff;
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  const TileLayout& L = P.L;
  fence_async_smem();
  __syncwarp();
  const uint32_t abytes = with_acts ? 32u * (uint32_t)(n + 1) : 0u;
  if (lane == 0) mbar_expect_tx(wb.a, (uint32_t)n * (768u + 64u + 32u) + abytes);
  for (int i = lane >> 1; i < n; i += 16) {
    const int64_t e = (int64_t)i * ld + b0;
    const uint32_t s = t + L.ports + i * 768;
    if (lane & 1) {
      bulk_g2s(s, P.st.port_i + e, 256, wb.a);
      bulk_g2s(s + 256, P.st.port_soc + e, 256, wb.a);
    } else {
      bulk_g2s(s + 512, P.st.port_de + e, 256, wb.a);
      bulk_g2s(t + L.dtrem + i * 64, P.st.port_dtrem + e, 64, wb.a);
      bulk_g2s(t + L.meta + i * 32, P.st.port_meta + e, 32, wb.a);
    }
  }
  // 32 rows x (n+1) bytes; the host guarantees a 16-byte aligned block and
  // that reading the whole block of a ragged last tile stays inside the allocation
  if (with_acts && lane == 31)
    bulk_g2s(t + L.acts, reinterpret_cast<const uint8_t*>(P.actions) + b0 * (n + 1), abytes, wb.a);
  wb.armed = true;
}

// Two-stage tile load (step kernel): the meta bytes (and action rows) first;
// once they arrive the warp votes which ports any of its 32 envs occupies and
// copies the float64 slots and dwell times of those ports only.  A port empty
// in every lane is never read (its slots are not used: phase 1 zeroes its
// current slot, phase 2 stages +0 obs and does not store it).
__device__ __forceinline__ void tile_issue_meta(const Params& P, uint32_t toff, int64_t b0, int lane,
                                                bool with_acts, WarpBar& wb) {
  const uint32_t t = smem_base() + toff;
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  const TileLayout& L = P.L;
  fence_async_smem();
  __syncwarp();
  const uint32_t abytes = with_acts ? 32u * (uint32_t)(n + 1) : 0u;
#if VY_BULK_META
  if (lane == 0) mbar_expect_tx(wb.a, 32u * (uint32_t)n + abytes);
  for (int c = lane; c < n; c += 32) bulk_g2s(t + L.meta + c * 32, P.st.port_meta + (int64_t)c * ld + b0, 32, wb.a);
  if (with_acts && lane == 31)
    bulk_g2s(t + L.acts, reinterpret_cast<const uint8_t*>(P.actions) + b0 * (n + 1), abytes, wb.a);
  wb.armed = true;
#else
  const char* msrc = reinterpret_cast<const char*>(P.st.port_meta);
  for (int c = lane >> 1; c < n; c += 16)
    cp_async16(t + L.meta + c * 32 + (lane & 1) * 16, msrc + ((int64_t)c * ld + b0) + (lane & 1) * 16);
  if (with_acts) {
    const char* asrc = reinterpret_cast<const char*>(P.actions) + b0 * (n + 1);
    for (int o = lane * 16; o < (int)abytes; o += 512) cp_async16(t + L.acts + o, asrc + o);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
#endif
}

// warp-uniform mask of the ports any env of the tile occupies (meta staged):
// port c's 32 meta bytes are words 8c..8c+7 of the meta area, word w is read
// by lane w % 32 in round w / 32
__device__ __forceinline__ uint64_t occupied_ports(const Params& P, uint32_t toff, int lane) {
  const int n = P.n_ports;
  const uint32_t* mw = reinterpret_cast<const uint32_t*>(vy_smem + toff + P.L.meta);
  uint64_t mask = 0;
  for (int r = 0; r * 32 < 8 * n; ++r) {
    const int w = r * 32 + lane;
    const bool occ = w < 8 * n && (mw[w] & 0x01010101u);
    const uint32_t bal = __ballot_sync(0xffffffffu, occ);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (bal & (0xFFu << (8 * q))) mask |= 1ull << (4 * r + q);
  }
  return mask;
}

// after tile_issue_meta: wait for the meta bytes, vote the occupied ports and
// issue their slot copies; returns the warp-uniform port mask
__device__ __forceinline__ uint64_t tile_issue_ports(const Params& P, uint32_t toff, int64_t b0, int lane,
                                                     WarpBar& wb, bool stream = false) {
#if VY_BULK_META
  bar_wait(wb);
#else
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncwarp();
#endif
  const uint32_t t = smem_base() + toff;
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  const TileLayout& L = P.L;
  const uint64_t mask = occupied_ports(P, toff, lane);
#if !VY_BULK_SLOTS
  const int q16 = (lane & 15) * 16;
  if (stream) {  // streamed tile: the i_drawn slots only (soc / de / dwell are read in the port loops)
    for (int i = lane >> 4; i < n; i += 2) {
      if (!((mask >> i) & 1ull)) continue;
      cp_async16(t + L.ports + i * 256 + q16, reinterpret_cast<const char*>(P.st.port_i) + ((int64_t)i * ld + b0) * 8 + q16);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    return mask;
  }
  for (int i = lane >> 4; i < n; i += 2) {
    if (!((mask >> i) & 1ull)) continue;
    const int64_t g = ((int64_t)i * ld + b0) * 8 + q16;
    const uint32_t d = t + L.ports + i * 768 + q16;
    cp_async16(d, reinterpret_cast<const char*>(P.st.port_i) + g);
    cp_async16(d + 256, reinterpret_cast<const char*>(P.st.port_soc) + g);
    cp_async16(d + 512, reinterpret_cast<const char*>(P.st.port_de) + g);
  }
  const char* dsrc = reinterpret_cast<const char*>(P.st.port_dtrem);
  for (int c = lane >> 2; c < n; c += 8)
    if ((mask >> c) & 1ull)
      cp_async16(t + L.dtrem + c * 64 + (lane & 3) * 16, dsrc + ((int64_t)c * ld + b0) * 2 + (lane & 3) * 16);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  return mask;
#endif
  if (mask) {
    if (lane == 0) mbar_expect_tx(wb.a, (uint32_t)__popcll(mask) * (768u + 64u));
    for (int i = lane >> 1; i < n; i += 16) {
      if (!((mask >> i) & 1ull)) continue;
      const int64_t e = (int64_t)i * ld + b0;
      const uint32_t s = t + L.ports + i * 768;
      if (lane & 1) {
        bulk_g2s(s, P.st.port_i + e, 256, wb.a);
        bulk_g2s(s + 256, P.st.port_soc + e, 256, wb.a);
      } else {
        bulk_g2s(s + 512, P.st.port_de + e, 256, wb.a);
        bulk_g2s(t + L.dtrem + i * 64, P.st.port_dtrem + e, 64, wb.a);
      }
    }
    wb.armed = true;
  }
  return mask;
}

// L2 prefetch (TMA engine: no shared memory, no registers held) of the state
// a later tile will read: its meta and per-env scalars, and the float64 slots
// and dwell times of the ports in `mask` (this tile's occupied ports; tiles at
// the same step have similar occupancy).  The persistent grid claims tiles in
// increasing order, so tile t + pf_dist is claimed a fraction of a tile
// lifetime later and its state loads then hit L2.  Used by the streamed tile
// (Spec<4>, config C4), whose in-loop state loads wait on memory latency with
// the DRAM system mostly idle; the resident-tile step is bound by DRAM
// throughput and measured slower with it (profiles/r2_l2_prefetch_ab.txt).
__device__ __forceinline__ void l2_prefetch(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tile_prefetch_l2(const Params& P, int64_t bp0, int lane, uint64_t mask, bool battery) {
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  const vy_state& s = P.st;
  for (int i = lane; i < n; i += 32) {
    const int64_t e = (int64_t)i * ld + bp0;
    l2_prefetch(s.port_meta + e, 32);
    if ((mask >> i) & 1ull) {
      l2_prefetch(s.port_i + e, 256);
      l2_prefetch(s.port_soc + e, 256);
      l2_prefetch(s.port_de + e, 256);
      l2_prefetch(s.port_dtrem + e, 64);
    }
  }
  const int j = 31 - lane;  // the per-env scalars from the top lanes
  if (j < 10 || (battery && j < 12)) {
    const void* a = j == 0 ? (const void*)(s.step + bp0) : j == 1 ? (const void*)(s.day + bp0)
                  : j == 2 ? (const void*)(s.akey + bp0) : j == 3 ? (const void*)(s.ep_profit + bp0)
                  : j == 4 ? (const void*)(s.ep_reward + bp0) : j == 5 ? (const void*)(s.ep_missing + bp0)
                  : j == 6 ? (const void*)(s.ep_energy + bp0) : j == 7 ? (const void*)(s.ep_overtime + bp0)
                  : j == 8 ? (const void*)(s.ep_declined + bp0) : j == 9 ? (const void*)(s.ep_departures + bp0)
                  : j == 10 ? (const void*)(s.b_i + bp0) : (const void*)(s.b_soc + bp0);
    const bool wide = (j >= 2 && j <= 6) || j >= 10;
    l2_prefetch(a, wide ? 256u : 128u);
  }
}

__device__ __forceinline__ void tile_wait(WarpBar& wb) {
  bar_wait(wb);
#if !VY_BULK_SLOTS || !VY_BULK_META
  cp_async_wait_all();
  __syncwarp();
#endif
}

template <int M>
__device__ __forceinline__ void load_env(const Params& P, int64_t b, EnvRegs& E) {
  using C = Spec<M>;
  const vy_state& s = P.st;
  E.step = ldg_s32(s.step + b);
  E.day = ldg_s32(s.day + b);
  E.akey = ldg_u64(s.akey + b);
  E.b_i = C::battery(P) ? ldg_f64(s.b_i + b) : 0.0;
  E.b_soc = C::battery(P) ? ldg_f64(s.b_soc + b) : 0.0;
  E.ep_profit = ldg_f64(s.ep_profit + b);
  E.ep_reward = ldg_f64(s.ep_reward + b);
  E.ep_missing = ldg_f64(s.ep_missing + b);
  E.ep_energy = ldg_f64(s.ep_energy + b);
  E.ep_overtime = ldg_s32(s.ep_overtime + b);
  E.ep_declined = ldg_s32(s.ep_declined + b);
  E.ep_departures = ldg_s32(s.ep_departures + b);
}

template <int M>
__device__ __forceinline__ void store_env(const Params& P, int64_t b, const EnvRegs& E, bool reset_too) {
  const vy_state& s = P.st;
  s.step[b] = E.step;
  if (Spec<M>::battery(P)) {
    s.b_i[b] = E.b_i;
    s.b_soc[b] = E.b_soc;
  }
  s.ep_profit[b] = E.ep_profit;
  s.ep_reward[b] = E.ep_reward;
  s.ep_missing[b] = E.ep_missing;
  s.ep_energy[b] = E.ep_energy;
  s.ep_overtime[b] = E.ep_overtime;
  s.ep_declined[b] = E.ep_declined;
  s.ep_departures[b] = E.ep_departures;
  if (reset_too) {
    s.day[b] = E.day;
    s.akey[b] = E.akey;
  }
}

// charge envelope (vehicles.py:22-35): rbar below tau, then (1-soc)*rbar/(1-tau)
__device__ __forceinline__ double envelope(double soc, double tau, double omt, double rcp_omt, double rbar) {
  const double taper = div_rcp((1.0 - soc) * rbar, omt, rcp_omt);  // five fp64 ops: cheaper than a branch
  return soc <= tau ? rbar : taper;
}

// Clip a requested current (_kernel.pyx:309-325 ports, :329-345 battery).  Charging
// is bounded by rhat = envelope(soc) (the value the reference stores,
// _kernel.pyx:389/505), discharging by envelope(1 - soc); one select-based path.
__device__ __forceinline__ double clip_current(double tgt, double soc, double tau, double omt, double rcp_omt,
                                               double rbar, double volt, double rcp_volt, double imax_c,
                                               double imax_d) {
  const bool chg = tgt >= 0.0;
  const double s = chg ? soc : 1.0 - soc;
  const double r = envelope(s, tau, omt, rcp_omt, rbar);
  const double lim = div_rcp(1000.0 * r, volt, rcp_volt);
  double v = chg ? tgt : -tgt;
  if (lim < v) v = lim;
  const double pm = chg ? imax_c : imax_d;
  if (pm < v) v = pm;
  return chg ? v : -v;
}

__device__ __forceinline__ double node_load(double s, double eta, double rcp_eta) {
  if (s > 0.0) return eta == 1.0 ? s : div_rcp(s, eta, rcp_eta);
  return s * eta;
}
__device__ __forceinline__ double node_load(const Params& P, double s, int m) {
  return node_load(s, P.node_eta[m], P.node_rcp_eta[m]);
}

// a node's load sum over its slot range [lo, hi), sequentially in leaf order
__device__ __forceinline__ double node_sum(const Params& P, const Lane& T, double cb, int lo, int hi) {
  const int hp = hi < P.n_ports ? hi : P.n_ports;
  double s = 0.0;
  for (int j = lo; j < hp; ++j) s += T.idr(j);
  if (P.battery && lo <= P.n_ports && P.n_ports < hi) s += cb;
  return s;
}

// _kernel.pyx:626-649: deepest-first proportional scaling to a fixed point.
// Currents live in the i_drawn slots (they become i_drawn after the rescale).
// `clean` (trees of at most 64 nodes): bit q set = node q's leaves are
// unchanged since it was last evaluated and that evaluation changed nothing,
// so evaluating it again is a no-op and is skipped.  A node whose rescale
// moves a current clears the bit of every node sharing a slot with it
// (itself included).  The values, the pass in which the loop stops and the
// max_passes bound are exactly the reference's: only no-op evaluations go.
// The caller seeds `clean` with the nodes its excess check found within
// capacity.
__device__ __noinline__ void fit_tree(const Params& P, TreeC tc, const Lane& T, double& cb, uint64_t clean) {
  const bool track = P.n_nodes <= 64;
  if (!track) clean = 0;
  for (int pass = 0; pass < P.max_passes; ++pass) {
    bool moved = false;
    for (int q = 0; q < P.n_nodes; ++q) {
      if ((clean >> q) & 1ull) continue;
      double cap, eta, rcp_eta;
      int lo, hi;
      tc.rec(q, cap, eta, rcp_eta, lo, hi);
      const double mag = fabs(node_load(node_sum(P, T, cb, lo, hi), eta, rcp_eta));
      bool mq = false;
      if (mag > cap) {
        const double f = cap / mag;
        const int hp = hi < P.n_ports ? hi : P.n_ports;
        for (int j = lo; j < hp; ++j) {
          const double old = T.idr(j);
          const double v = old * f;
          if (v != old) {
            T.idr(j) = v;
            mq = true;
          }
        }
        if (P.battery && lo <= P.n_ports && P.n_ports < hi) {
          const double v = cb * f;
          if (v != cb) {
            cb = v;
            mq = true;
          }
        }
      }
      if (!track) {
        moved |= mq;
      } else if (mq) {
        moved = true;
        for (int r = 0; r < P.n_nodes; ++r) {
          double c2, e2, re2;
          int lo2, hi2;
          tc.rec(r, c2, e2, re2, lo2, hi2);
          if (lo2 < hi && lo < hi2) clean &= ~(1ull << r);
        }
      } else {
        clean |= 1ull << q;
      }
    }
    if (!moved) return;
  }
}

// reset_env (_kernel.pyx:239-261), scalar part: draw the day, zero the clock
// and the episode accumulators, re-initialise the battery.  The caller clears
// the ports (tile slots, or HBM + obs staging when the slots hold obs).
__device__ __forceinline__ void reset_scalars(const Params& P, EnvRegs& E, uint64_t seed, int episode, int inj_day,
                                              bool use_inj) {
  uint64_t st = fold(fold(fold(fold(kKey0, seed), (uint64_t)(int64_t)episode), 0), 0);
  E.day = use_inj ? inj_day : below(st, P.n_days);
  E.step = 0;
  E.akey = fold(fold(fold(kKey0, seed), (uint64_t)(int64_t)episode), 1);
  E.b_soc = P.battery ? P.b_init_soc : 0.0;
  E.b_i = 0.0;
  E.ep_profit = E.ep_reward = E.ep_missing = E.ep_energy = 0.0;
  E.ep_overtime = E.ep_declined = E.ep_departures = 0;
}

__device__ __forceinline__ void clear_tile_ports(const Params& P, const Lane& T) {
  for (int i = 0; i < P.n_ports; ++i) {
    T.idr(i) = 0.0;
    T.soc(i) = 0.0;
    T.de(i) = 0.0;
    T.dtrem(i) = 0;
    T.meta(i) = 0;
  }
}

struct StepResult {
  double reward;
  bool done;
};

// eff_day = (day + t*dt_min // 1440) % n_days (_kernel.pyx:290) in 32-bit
// integers (t*dt_min < 32000 * 1440: vy_create bounds the episode) with the
// constant divisors strength-reduced; the runtime modulo only when the day
// wraps (0 <= day < n_days)
__device__ __forceinline__ int effective_day(const Params& P, int t, int day) {
  int eff = day + t * P.dt_min / 1440;
  if (eff >= P.n_days) eff %= P.n_days;
  return eff;
}

// Exogenous inputs of the step at (step, day) (_kernel.pyx:289-295), loaded
// before the tile's cp.async copies are awaited so their latency overlaps.
struct Frame {
  double p_buy, p_sg, moer, dgrid, pthr;
  int hidx, lam_idx, pfull;
};
template <int M>
__device__ __forceinline__ Frame load_frame(const Params& P, int t, int day) {
  Frame F;
  const int eff_day = effective_day(P, t, day);
  F.hidx = eff_day * 24 + (t * P.dt_min / 60) % 24;
  F.p_buy = ldg_nc_f64(P.buy + F.hidx);
  F.p_sg = ldg_nc_f64(P.sellg + F.hidx);
  F.moer = Spec<M>::moer(P) ? ldg_nc_f64(P.moer + F.hidx) : 0.0;
  F.dgrid = Spec<M>::dgrid(P) ? ldg_nc_f64(P.dgrid + F.hidx) : 0.0;
  F.lam_idx = (ldg_nc_s8(P.weekday + eff_day) ? 0 : P.lam_len) + (t < P.lam_len ? t : t % P.lam_len);
  F.pfull = ldg_nc_s32(P.pois_full + F.lam_idx);
  F.pthr = ldg_nc_f64(P.pois_thr + F.lam_idx);
  return F;
}

// Observation globals at (step, day) (_kernel.pyx:577-603): buy, sellg, sin, cos,
// weekday, day/365 — prefetched for step t+1 at the start of the step.
struct ObsGlobals {
  double buy, sellg, sinv, cosv, wk, dayf;
  int step, day;
};
__device__ __forceinline__ ObsGlobals load_obs_globals(const Params& P, int step, int day) {
  ObsGlobals G;
  const int eff_day = effective_day(P, step, day);
  const int hidx = eff_day * 24 + (step * P.dt_min / 60) % 24;
  const int sod = step < P.steps_per_day ? step : step % P.steps_per_day;
  G.buy = ldg_nc_f64(P.buy + hidx);
  G.sellg = ldg_nc_f64(P.sellg + hidx);
  G.sinv = ldg_nc_f64(P.sin_t + sod);
  G.cosv = ldg_nc_f64(P.cos_t + sod);
  G.wk = (double)ldg_nc_s8(P.weekday + eff_day);
  G.dayf = div_rcp((double)eff_day, 365.0, P.rcp_365);
  G.step = step;
  G.day = day;
  return G;
}

// Where a step's outputs go.  f32 obs are staged column-major in shared
// memory at `cells` (column c, row r at cells + c*132 + r*4: per-lane writes and
// per-row reads are both bank-conflict free) and leave with coalesced row-major
// stores; f64 obs (exact drop-in mode) go straight to this lane's row.  With
// `in_place` the staging area is the tile's own float64 port slots: port i's
// state is written to HBM, then its slots take its obs columns (the 24n-byte
// pad in front of the slots makes column block 6i..6i+5 end before port i+1).
struct ObsSink {
  uint32_t cells;
  double* row64;
  bool in_place;
  // Rollout ("chunk") mode: no whole-tile staging area.  Each port's six
  // columns go through a two-port ring of 6-column buffers (column stride
  // kChunkCol words) and leave right away: lane l stores column l % 6 of rows
  // l / 6 + 5k (k = 0..6), 24-byte row segments the L2 merges into whole
  // sectors.  The smem a tile needs drops from 132 * obs_len bytes to
  // 2 * 6 * 4 * kChunkCol, so more warps fit per SM.
  bool chunk;
  float* gtile;  // chunk: f32 obs row 0 of the tile
  float* glane;  // chunk: this lane's read-out cell of port 0: row l / 6, column l % 6
  uint32_t soff; // chunk: byte offset of that cell in a ring buffer
  int s5;        // chunk: 5 * obs_len (5 rows per read-out pass)
  int rows;      // chunk: live rows of the tile
};
// column stride of the chunk buffers in 4-byte words: 37 = 5 mod 32, so the
// read-out's (column f, row r) words 37f + r hit distinct banks for f < 6, r < 5
constexpr int kChunkCol = 37;
constexpr int kChunkBuf = 6 * kChunkCol * 4;  // bytes per 6-column buffer
// VY_RING1 (default): one 6-column buffer (a second __syncwarp per port) and
// the tail columns stored from registers by each lane, so a rollout tile
// fits 15 warps per SM instead of 14 (rollout -2.8%, streamed C4 -4.8% step
// time against the two-buffer ring, profiles/r2_ring_ab.txt)
#ifndef VY_RING1
#define VY_RING1 1
#endif
constexpr int kRingBufs = VY_RING1 ? 1 : 2;

// chunk mode: coalesced read-out of port i's 6 staged columns (ring buffer
// `buf`) into global obs columns [6i, 6i + 6): lanes 0..29 store rows l / 6 +
// 5k, column l % 6 (k = 0..6; rows 30, 31 by lanes 0..11)
__device__ __forceinline__ void chunk_out6(const ObsSink& S, int lane, uint32_t buf, int i) {
  if (lane >= 30) return;
  float* g = S.glane + 6 * i;
  const uint32_t a = buf + S.soff;
  if (S.rows == 32 && S.s5 == 5 * 105) {
    // the 16-port station (obs_len 105): row offsets are immediates of the stores
#pragma unroll
    for (int k = 0; k < 6; ++k) __stcs(g + 525 * k, lds_f32(a + 20 * k));
    if (lane < 12) __stcs(g + 3150, lds_f32(a + 120));
  } else if (S.rows == 32) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      __stcs(g, lds_f32(a + 20 * k));
      g += S.s5;
    }
    if (lane < 12) __stcs(g, lds_f32(a + 120));
  } else {
    const int r0 = lane / 6;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      if (r0 + 5 * k < S.rows) __stcs(g, lds_f32(a + 20 * k));
      g += S.s5;
    }
  }
}
// chunk mode: +0 into port i's obs columns of the rows in `rowmask`
__device__ __forceinline__ void chunk_zero6(const ObsSink& S, int lane, int i, uint32_t rowmask) {
  if (lane >= 30) return;
  float* g = S.glane + 6 * i;
  const int r0 = lane / 6;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const int r = r0 + 5 * k;
    if (r < S.rows && ((rowmask >> r) & 1u)) __stcs(g, 0.0f);
    g += S.s5;
  }
}

__device__ __forceinline__ void stage_port_obs(const Params& P, Prof prof, const ObsSink& S, int lane,
                                               bool active, int i, uint32_t mt, double idr, double soc, double de,
                                               int dt, double i_denom, double rcp_i_denom, bool own_row = false) {
  const bool occ = mt & 1u;
  double v[6];
  v[0] = occ ? 1.0 : 0.0;
  v[1] = div_rcp(idr, i_denom, rcp_i_denom);
  v[2] = soc;
  const double dec = div_rcp(de, prof.cap(mt >> 2), prof.rcp_cap(mt >> 2));  // empty port: 0/cap0, discarded
  v[3] = occ ? dec : 0.0;
  v[4] = div_rcp((double)dt, (double)P.episode_steps, P.rcp_ep);
  v[5] = (double)((mt >> 1) & 1u);
  if (S.row64) {
    if (active)
#pragma unroll
      for (int f = 0; f < 6; ++f) S.row64[6 * i + f] = v[f];
  } else if (S.chunk) {
    if (own_row) {  // a single lane's port (arrivals): its own row, directly
      if (active)
#pragma unroll
        for (int f = 0; f < 6; ++f) S.gtile[(int64_t)lane * P.obs_len + 6 * i + f] = (float)v[f];
    } else {
      const uint32_t buf = S.cells + (kRingBufs == 2 ? (i & 1) * kChunkBuf : 0);
#pragma unroll
      for (int f = 0; f < 6; ++f) sts_f32(buf + f * (kChunkCol * 4) + lane * 4, (float)v[f]);
      __syncwarp();  // also orders the read-out of port i - 1 (other buffer) before port i + 1 reuses it
      chunk_out6(S, lane, buf, i);
      if (kRingBufs == 1) __syncwarp();  // one buffer: read out before the next port stages
    }
  } else {
    const uint32_t col = S.cells + 6 * i * 132 + lane * 4;
#pragma unroll
    for (int f = 0; f < 6; ++f) sts_f32(col + f * 132, (float)v[f]);
  }
}

// the six obs columns of a port that is empty (all-zero state): +0
__device__ __forceinline__ void stage_zero_obs(const Params& P, const ObsSink& S, int lane, bool active, int i) {
  if (S.row64) {
    if (active)
#pragma unroll
      for (int f = 0; f < 6; ++f) S.row64[6 * i + f] = 0.0;
  } else if (S.chunk) {
    chunk_zero6(S, lane, i, 0xffffffffu);
  } else {
    const uint32_t col = S.cells + 6 * i * 132 + lane * 4;
#pragma unroll
    for (int f = 0; f < 6; ++f) sts_f32(col + f * 132, 0.0f);
  }
}

__device__ __forceinline__ void store_port(const Params& P, int64_t b, int i, uint32_t mt, double idr, double soc,
                                           double de, int dt, bool meta = true) {
  const vy_state& s = P.st;
  const int64_t e = (int64_t)i * P.ld + b;
  s.port_i[e] = idr;
  s.port_soc[e] = soc;
  s.port_de[e] = de;
  s.port_dtrem[e] = (int16_t)dt;
  if (meta) s.port_meta[e] = (uint8_t)mt;  // callers skip it when unchanged
}

// One transition of one env (_kernel.pyx:283-571).  `act(slot)` returns the
// action index of a slot; `b` is the global env index (infos / injected draws).
// U2: unroll factor of the charge/departure port loop.  1 for the single step
// (rolled: its hot loop is smaller; 2 measured 6% slower, the step being bound
// by DRAM); 2 for the rollout, which is latency-bound with its state resident
// and gains from the two ports' independent float64 chains (-1.8% per step,
// profiles/r2_unroll_ab.txt).
template <int M, class Act, int U2 = 1>
__device__ __forceinline__ StepResult tile_step(const Params& P, Prof prof,
                                                const double* __restrict__ dtab, PortC pc, TreeC tc, const Lane& T,
                                                EnvRegs& E, int64_t b, const Frame& F, const ObsSink& S, bool active,
                                                Act act, const uint64_t* occ_ports) {
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  using C = Spec<M>;
  const bool info = C::info(P);
  const bool battery = C::battery(P);
  const vy_outputs& O = P.out;
  const int t = E.step;

  const double p_buy = F.p_buy, p_sg = F.p_sg;
  const int hidx = F.hidx;
  (void)hidx;

  // phase 1: apply actions (_kernel.pyx:297-356); the clipped current replaces
  // i_drawn in its smem slot, node loads accumulate in leaf order on the fly
  const int hi_a = 2 * P.k;
  // (a-k)/k: with 2k+1 <= 32 the grid lives one entry per lane and a warp
  // shuffle fetches it (a random-index shared-memory lookup bank-conflicts);
  // otherwise the staged table, else the IEEE division.
  const bool shfl_grid = C::lean || (hi_a < 32 && dtab);
  const double grid_lane = shfl_grid ? dtab[T.lane <= hi_a ? T.lane : 0] : 0.0;
  // out-of-range actions are clamped and flagged once per step (lazy error word)
  bool bad_action = false;
  auto delta_of = [&](int a) -> double {
    bad_action |= (unsigned)a > (unsigned)hi_a;
    a = min(max(a, 0), hi_a);
    if (shfl_grid) return __shfl_sync(0xffffffffu, grid_lane, a);
    return dtab ? dtab[a] : (double)(a - P.k) / (double)P.k;
  };
  const bool fast = C::fast_tree(P);
  double nsum[kFastNodes];
#pragma unroll
  for (int m = 0; m < kFastNodes; ++m) nsum[m] = 0.0;
  // streamed tile: soc of port i + 2 is requested while port i is worked on (3 ahead measured 4% slower: registers)
  const uint64_t occ_mask = occ_ports ? *occ_ports : ~0ull;
  auto soc_at = [&](int i) -> double {
    return i < n && ((occ_mask >> i) & 1ull) ? ldg_st_f64(P.st.port_soc + (int64_t)i * ld + b) : 0.0;
  };
  double soc_q0 = 0.0, soc_q1 = 0.0;
  if (C::stream) {
    soc_q0 = soc_at(0);
    soc_q1 = soc_at(1);
  }
#pragma unroll 1  // rolled: smaller hot loop measured faster than unroll 2 or 4
  for (int i = 0; i < n; ++i) {
    const double d = delta_of(act(i));
    const uint32_t mt = T.meta(i);
    const double idr_i = T.idr(i);
    double soc_i;
    if (C::stream) {
      soc_i = soc_q0;
      soc_q0 = soc_q1;
      soc_q1 = soc_at(i + 2);
    } else {
      soc_i = T.soc(i);
    }
    // A port no lane of the warp occupies is skipped (a bit of the tile's
    // warp-uniform port mask, one uniform branch); otherwise branch-free: an
    // empty port (meta 0 -> profile 0, zero slots) runs the same arithmetic
    // and the select discards it.
    double c = 0.0;
    double kind_nodes[2];
    pc.pair(i, 2, kind_nodes[0], kind_nodes[1]);
    // some lane occupies port i: the tile's warp-uniform port mask when the
    // caller has one (step kernel), else a vote (rollout)
    if (occ_ports ? (*occ_ports >> i) & 1ull : __any_sync(0xffffffffu, mt & 1u)) {
      double imax_c, imax_d, volt, rcp_volt;
      pc.pair(i, 0, imax_c, imax_d);
      pc.pair(i, 1, volt, rcp_volt);
      double tgt = idr_i + d * imax_c;
      if (!P.allow_discharge && tgt < 0.0) tgt = 0.0;
      const int pf = mt >> 2;
      c = clip_current(tgt, soc_i, prof.tau(pf), prof.omt(pf), prof.rcp_omt(pf),
                       kind_nodes[0] != 0.0 ? prof.r_dc(pf) : prof.r_ac(pf), volt, rcp_volt, imax_c, imax_d);
      c = (mt & 1u) ? c : 0.0;
    }
    T.idr(i) = c;
    if (info) O.i_att[i * ld + b] = c;
    const uint32_t pm = (uint32_t)kind_nodes[1];
#pragma unroll
    for (int m = 0; m < kFastNodes; ++m)
      if (pm & (1u << m)) nsum[m] += c;
  }
  double cb = 0.0;
  {
    // the battery slot is validated even when the battery is disabled (engine.py:440-442)
    const double d = delta_of(act(n));
    if (battery) {
      const double tgt = E.b_i + d * P.b_imax;
      cb = clip_current(tgt, E.b_soc, P.b_tau, P.b_omt, P.b_rcp_omt, P.b_rmax, P.b_volt, P.b_rcp_volt, P.b_imax,
                        P.b_imax);
      if (info) O.i_att[n * ld + b] = cb;
#pragma unroll
      for (int m = 0; m < kFastNodes; ++m)
        if (P.battery_node_mask & (1 << m)) nsum[m] += cb;
    }
  }
  if (bad_action) atomicOr(P.err, 1u);
  // tree: excess on the requested currents (_kernel.pyx:611-624), then rescale
  double excess = 0.0;
  uint64_t clean = 0;  // nodes the excess check found within capacity (fit_tree)
  if (fast) {
#pragma unroll
    for (int m = 0; m < kFastNodes; ++m) {
      if (m < P.n_nodes) {
        const double over = fabs(node_load(P, nsum[m], m)) - P.node_cap[m];
        if (over > excess) excess = over;
      }
    }
  } else {
    for (int q = 0; q < P.n_nodes; ++q) {  // max over the nodes: any order
      double cap, eta, rcp_eta;
      int lo, hi;
      tc.rec(q, cap, eta, rcp_eta, lo, hi);
      const double over = fabs(node_load(node_sum(P, T, cb, lo, hi), eta, rcp_eta)) - cap;
      if (over > excess) excess = over;
      if (!(over > 0.0)) clean |= 1ull << (q & 63);  // within capacity (mag <= cap)
    }
  }
  // no node over capacity => the reference's first rescale pass changes nothing and returns
  if (excess > 0.0) fit_tree(P, tc, T, cb, clean);
  if (info) {
    for (int i = 0; i < n; ++i) O.i_used[i * ld + b] = T.idr(i);
    if (battery) O.i_used[n * ld + b] = cb;
  }
  if (battery) E.b_i = cb;

  // phases 2+3: charge (_kernel.pyx:358-424), dwell countdown (:420-422) and
  // departures (:426-458) fused into one pass in port order; the same pass
  // emits each port's final state (HBM, or the resident tile) and its obs
  // columns.  Arrivals below patch the few ports that receive a car.
  double e_net = 0.0, e_in = 0.0, e_out = 0.0;
  double sat0 = 0.0, sat1 = 0.0;
  int nd = 0, tover = 0;
  uint64_t occm = 0;
  const bool last = t + 1 == P.episode_steps;
  // streamed tile: soc / de / dwell of port i + 2 requested while port i is worked on
  struct PortQ {
    double soc, de;
    int dt;
  };
  auto q_at = [&](int i) -> PortQ {
    if (i < n && ((occ_mask >> i) & 1ull)) {
      const int64_t e = (int64_t)i * ld + b;
      return {ldg_st_f64(P.st.port_soc + e), ldg_st_f64(P.st.port_de + e), ldg_st_s16(P.st.port_dtrem + e)};
    }
    return {0.0, 0.0, 0};
  };
  PortQ q0{0.0, 0.0, 0}, q1{0.0, 0.0, 0};
  if (C::stream) {
    q0 = q_at(0);
    q1 = q_at(1);
  }
#pragma unroll U2
  for (int i = 0; i < n; ++i) {
    uint32_t mt = T.meta(i);
    double cur = T.idr(i), soc, de;
    int dt;
    if (C::stream) {
      soc = q0.soc, de = q0.de, dt = q0.dt;
      q0 = q1;
      q1 = q_at(i + 2);
    } else {
      soc = T.soc(i), de = T.de(i), dt = T.dtrem(i);
    }
    // Ports no lane of the warp occupies are skipped (port mask, uniform
    // branch).  Otherwise branch-free: an empty port holds meta 0 and zero
    // slots, its current is 0 (phase 1), so the arithmetic below yields
    // got = +0, soc = de = 0 for it; only the dwell countdown and the
    // departure test are gated.  Sums that start at +0 never become -0, so
    // the +0 terms of empty / staying ports leave them bit-identical to the
    // reference's conditional adds.
    const bool occ = mt & 1u;
    double got = 0.0;
    bool dep = false;
    const bool any_occ = occ_ports ? (*occ_ports >> i) & 1ull : __any_sync(0xffffffffu, occ);  // meta unchanged since phase 1
    if (any_occ) {
      const int pf = mt >> 2;
      double dtv, eta_d, eta_c, rcp_eta_c;
      pc.pair(i, 3, dtv, eta_d);
      pc.pair(i, 4, eta_c, rcp_eta_c);
      const double raw = div_rcp(dtv * cur, 1000.0, P.rcp_1000);
      {
        double gc = raw;
        if (de < gc) gc = de;
        const double room = prof.cap(pf) * (1.0 - soc);
        if (room < gc) gc = room;
        const double fl = -prof.cap(pf) * soc;
        const double gd = raw < fl ? fl : raw;
        got = raw >= 0.0 ? gc : gd;
      }
      soc = soc + div_rcp(got, prof.cap(pf), prof.rcp_cap(pf));
      soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
      de = de - got;
      de = de < 0.0 ? 0.0 : de;
      e_net += got;
      const double gin = eta_c == 1.0 ? got : div_rcp(got, eta_c, rcp_eta_c);
      e_in += got > 0.0 ? gin : 0.0;
      e_out += got < 0.0 ? got * eta_d : 0.0;
      dt -= occ ? 1 : 0;
      const int p = (mt >> 1) & 1u;
      dep = occ & ((p == 0 & dt <= 0) | (p == 1 & de == 0.0));  // bitwise: no short-circuit branches
      // Departure bookkeeping (_kernel.pyx:426-458) behind a warp vote: about
      // 1.3% of occupied port-steps depart, so most warps skip it; lanes of a
      // voting warp without a departure add +0 (sums that start at +0 never
      // become -0, so that equals the reference's skipped add).
      if (__any_sync(0xffffffffu, dep)) {
        const int over = dt < 0 ? -dt : 0, early = dt > 0 ? dt : 0;
        if (info && dep) {
          const int64_t at = (int64_t)nd * ld + b;
          O.dep_port[at] = i;
          O.dep_missing[at] = de;
          O.dep_overtime[at] = over;
          O.dep_early[at] = early;
          O.dep_pref[at] = p;
          O.dep_cap[at] = prof.cap(pf);
          O.dep_soc[at] = soc;
        }
        sat0 += dep & (p == 0) ? de : 0.0;
        const double s1 = (double)over - P.beta * (double)early;
        sat1 += dep & (p == 1) ? s1 : 0.0;
        E.ep_missing += dep ? de : 0.0;
        E.ep_overtime += dep ? over : 0;
        E.ep_departures += dep ? 1 : 0;
        nd += dep ? 1 : 0;
      }
      // _kernel.pyx:559-561 (arrivals add dt > 0 only): the episode's last step only
      if (last) tover += !dep & (p == 1) & (dt < 0) ? -dt : 0;
      occm |= (uint64_t)(occ && !dep) << i;
    }
    if (info) O.delivered[i * ld + b] = got;
    if (any_occ) {
      if (dep) {
        mt = 0;
        cur = soc = de = 0.0;
        dt = 0;
      }
      if (S.in_place) {
        // padding lanes (b >= B) write their own padding columns of the [n][ld] state: harmless, no branch;
        // the meta byte changes only on a departure
        store_port(P, b, i, mt, cur, soc, de, dt, dep);
        __syncwarp();  // every lane has read port i before its slots take obs columns
      } else {
        T.meta(i) = (uint8_t)mt;
        T.idr(i) = cur;
        T.soc(i) = soc;
        T.de(i) = de;
        T.dtrem(i) = (int16_t)dt;
      }
      double i_denom, rcp_i_denom;
      pc.pair(i, 5, i_denom, rcp_i_denom);
      stage_port_obs(P, prof, S, T.lane, active, i, mt, cur, soc, de, dt, i_denom, rcp_i_denom);
    } else {
      // A port empty in every lane of the warp stays empty and all-zero (a
      // departure or reset stored zeros, phase 1 set its current to 0): its
      // HBM copy already holds this state, so it is not rewritten, and its
      // six obs columns are +0.  Arrivals below store the ports they fill.
      if (S.in_place) __syncwarp();  // every lane has read port i before its slots take obs columns
      stage_zero_obs(P, S, T.lane, active, i);
    }
  }
  if (S.chunk) __syncwarp();  // the ports' read-outs land before arrivals rewrite their own rows
  double e_b = 0.0, bgot = 0.0;
  if (battery) {
    bgot = div_rcp(P.b_dtv * E.b_i, 1000.0, P.rcp_1000);
    if (bgot >= 0.0) {
      const double room = P.b_cap * (1.0 - E.b_soc);
      if (room < bgot) bgot = room;
    } else {
      const double fl = -P.b_cap * E.b_soc;
      if (bgot < fl) bgot = fl;
    }
    const double soc = E.b_soc + div_rcp(bgot, P.b_cap, P.b_rcp_cap);
    E.b_soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
    e_b = bgot > 0.0 ? div_rcp(bgot, P.b_eta_c, P.b_rcp_eta_c) : bgot * P.b_eta_d;
  }
  if (info) {
    O.b_delivered[b] = bgot;
    O.dep_n[b] = nd;
  }
  const double e_grid_net = e_in + e_out + e_b;

  // phase 4: arrivals (_kernel.pyx:460-509); draws of Stream(key4(seed, ep, 1, t))
  uint64_t st = fold(E.akey, (uint64_t)(int64_t)t);
  const bool inj = C::inject(P);
  int m = 0;
  int64_t inj0 = 0;
  if (inj) {
    if (active) {  // padding lanes have no draw rows
      inj0 = P.inj.off[b];
      m = P.inj.off[b + 1] - (int)inj0;
    }
  } else {
    const int full = F.pfull;
    if (full >= 0) {
      for (int c = 0; c < full; ++c) m += knuth(st, P.thr32);
      m += knuth(st, F.pthr);
    }
  }
  const int nfree = n - __popcll(occm);
  const int admitted = m < nfree ? m : nfree;
  const int declined = m - admitted;
  // Only the admitted cars (the first min(M, free) of the M arrivals) are
  // drawn: the declined cars' draws come after them in this step's own
  // stream key4(seed, ep, 1, t), which nothing else reads, so skipping them
  // changes no output (M and `declined` are counts).
  for (int j = 0; j < admitted; ++j) {
    int car, stay;
    double soc0, frac;
    uint32_t pref;
    if (inj) {
      car = P.inj.profile[inj0 + j];
      stay = P.inj.stay[inj0 + j];
      soc0 = P.inj.soc0[inj0 + j];
      frac = P.inj.frac[inj0 + j];
      pref = P.inj.pref[inj0 + j] ? 1u : 0u;
    } else {
      const double u = unit(st);
      car = P.n_cat - 1;
      for (int e = 0; e < P.n_cat - 1; ++e)
        if (u < prof.cum(e)) {
          car = e;
          break;
        }
      stay = P.stay_lo + below(st, P.stay_span);
      soc0 = P.soc_lo + unit(st) * P.soc_span;
      frac = P.frac_lo + unit(st) * P.frac_span;
      pref = unit(st) < P.p_charge ? 1u : 0u;
    }
    const uint64_t freem = ~occm & (n == 64 ? ~0ull : ((1ull << n) - 1));
    int port = 0;
    if (C::identity(P)) {
      port = __ffsll((long long)freem) - 1;
    } else {
      for (int q = 0; q < n; ++q)
        if ((freem >> P.order[q]) & 1ull) {
          port = P.order[q];
          break;
        }
    }
    occm |= 1ull << port;
    const uint32_t mt = 1u | (pref << 1) | ((uint32_t)car << 2);
    const double de0 = frac * prof.cap(car) * (1.0 - soc0);
    if (S.in_place) {
      store_port(P, b, port, mt, 0.0, soc0, de0, stay);
    } else {
      T.meta(port) = (uint8_t)mt;
      T.idr(port) = 0.0;
      T.soc(port) = soc0;
      T.de(port) = de0;
      T.dtrem(port) = (int16_t)stay;
    }
    // a new car draws no current yet: I / i_denom = 0 for any denominator
    stage_port_obs(P, prof, S, T.lane, active, port, mt, 0.0, soc0, de0, stay, 1.0, 1.0, /*own_row=*/true);
  }
  E.ep_declined += declined;
  if (info) {
    O.arrivals_m[b] = m;
    O.declined[b] = declined;
  }

  // reward (_kernel.pyx:511-551)
  const double price = e_grid_net > 0.0 ? p_buy : p_sg;
  const double profit = P.p_sell * e_net - price * e_grid_net - P.c_dt;
  double c[8];
  c[0] = excess;
  c[1] = sat0;
  c[2] = sat1;
  c[3] = C::moer(P) ? F.moer * e_grid_net : 0.0;
  c[4] = (double)declined;
  c[5] = e_b < 0.0 ? -e_b : 0.0;
  c[6] = e_out < 0.0 ? -e_out : 0.0;
  if (C::dgrid(P)) {
    const double d = e_net - F.dgrid;
    c[7] = d >= 0.0 ? d : -d;
  } else {
    c[7] = 0.0;
  }
  double reward = profit;
#pragma unroll
  for (int q = 0; q < 8; ++q) reward -= P.alphas[q] * c[q];
  if (info) {
    O.breakdown[b] = profit;
#pragma unroll
    for (int q = 0; q < 8; ++q) O.breakdown[(q + 1) * ld + b] = c[q];
    O.breakdown[9 * ld + b] = reward;
    O.flows[b] = e_net;
    O.flows[ld + b] = e_in;
    O.flows[2 * ld + b] = e_out;
    O.flows[3 * ld + b] = e_b;
    O.flows[4 * ld + b] = e_grid_net;
  }
  E.ep_profit += profit;
  E.ep_reward += reward;
  E.ep_energy += e_net;

  // advance (_kernel.pyx:553-570)
  E.step = t + 1;
  const bool done = t + 1 == P.episode_steps;
  if (done || info) {
    if (done) {
      double* es = O.ep_stats;
      es[b] = E.ep_profit;
      es[ld + b] = E.ep_reward;
      es[2 * ld + b] = E.ep_missing;
      es[3 * ld + b] = (double)E.ep_overtime;
      es[4 * ld + b] = (double)E.ep_declined;
      es[5 * ld + b] = E.ep_energy;
      es[6 * ld + b] = (double)E.ep_departures;
      es[7 * ld + b] = (double)tover;
    }
    O.term_overtime[b] = tover;
  }
  return {reward, done};
}

// ---- observation (_kernel.pyx:575-607; layout config.py:99-130) ----------------

__device__ __forceinline__ void bulk_s2g(void* gdst, uint32_t soff, uint32_t bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(vy_smem + soff);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// Write the tile's per-port state back to HBM with bulk async copies (the TMA
// engine streams each 256/64/32-byte column; no per-lane stores or 64-bit
// address math).  Padding lanes write their (unchanged) padding columns.
// Returns after the copies have finished READING shared memory, so the
// caller may overwrite the port slots.
__device__ __forceinline__ void tile_store(const Params& P, uint32_t toff, int64_t b0, int lane) {
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  fence_async_smem();  // make this warp's STS visible to the async proxy
  __syncwarp();
  for (int c = lane; c < 5 * n; c += 32) {
    const int i = c / 5, f = c - 5 * i;
    const int64_t e = (int64_t)i * ld + b0;
    if (f < 3) {
      double* g = f == 0 ? P.st.port_i : f == 1 ? P.st.port_soc : P.st.port_de;
      bulk_s2g(g + e, toff + P.L.ports + i * 768 + f * 256, 256);
    } else if (f == 3) {
      bulk_s2g(P.st.port_dtrem + e, toff + P.L.dtrem + i * 64, 64);
    } else {
      bulk_s2g(P.st.port_meta + e, toff + P.L.meta + i * 32, 32);
    }
  }
  bulk_commit();
  bulk_wait_read();
  __syncwarp();
}

template <int M>
__device__ __forceinline__ ObsSink make_sink(const Params& P, const Lane& T, int64_t b, void* obs_base,
                                             bool in_place) {
  ObsSink S;
  S.cells = smem_base() + T.t + P.L.obs;
  S.row64 = Spec<M>::f64(P) ? reinterpret_cast<double*>(obs_base) + b * P.obs_len : nullptr;
  S.in_place = in_place;
  S.chunk = false;
  S.gtile = nullptr;
  S.glane = nullptr;
  S.soff = 0;
  S.s5 = 0;
  S.rows = 0;
  return S;
}

// rollout sink: f32 obs through the per-port chunk ring (ObsSink::chunk), or
// f64 rows directly
template <int M>
__device__ __forceinline__ ObsSink make_chunk_sink(const Params& P, const Lane& T, int64_t b0, void* obs_base,
                                                   bool state_to_hbm = false) {
  ObsSink S = make_sink<M>(P, T, b0 + T.lane, obs_base, /*in_place=*/state_to_hbm);
  if (!S.row64) {
    S.chunk = true;
    S.gtile = reinterpret_cast<float*>(obs_base) + b0 * P.obs_len;
    const int64_t left = P.B - b0;
    S.rows = left >= 32 ? 32 : (int)left;
    const int rf = T.lane % 6, rr = T.lane / 6;
    S.glane = S.gtile + rr * P.obs_len + rf;
    S.soff = (uint32_t)(rf * (kChunkCol * 4) + rr * 4);
    S.s5 = 5 * P.obs_len;
  }
  return S;
}

// Global obs columns and the coalesced read-out of the staged [rows][OL] block.
template <int M>
__device__ __forceinline__ void emit_tail(const Params& P, const Lane& T, const EnvRegs& E, ObsGlobals G,
                                          const ObsSink& S, int64_t b0, bool active, void* obs_base) {
  const int n = P.n_ports;
  const int lane = T.lane;
  const int OL = P.obs_len;
  if (G.step != E.step || G.day != E.day) G = load_obs_globals(P, E.step, E.day);  // auto-reset happened
  // battery [soc, I/Imax], [buy, sellg, p_sell, sin, cos, weekday, day/365], price horizon
  double gv[9];
  gv[0] = E.b_soc;
  gv[1] = div_rcp(E.b_i, P.b_idenom, P.b_rcp_idenom);
  gv[2] = G.buy;
  gv[3] = G.sellg;
  gv[4] = P.p_sell;
  gv[5] = G.sinv;
  gv[6] = G.cosv;
  gv[7] = G.wk;
  gv[8] = G.dayf;
  const int c0 = 6 * n;
  // chunk mode: the tail columns are staged from column 0 of the chunk ring
  // (stride kChunkCol words) once every lane's earlier read-outs are done
  if (S.chunk) __syncwarp();
  if (S.chunk && kRingBufs == 1) {
    // single-buffer ring: each lane stores its own row's tail columns
    if (active) {
      float* row = S.gtile + (int64_t)lane * OL + c0;
#pragma unroll
      for (int k = 0; k < 9; ++k) __stcs(row + k, (float)gv[k]);
      for (int h = 0; h < Spec<M>::horizon(P); ++h) {
        const int64_t fmin = (int64_t)(E.step + 1 + h) * P.dt_min;
        const int64_t fday = ((int64_t)E.day + fmin / 1440) % P.n_days;
        __stcs(row + 9 + h, (float)__ldg(P.buy + fday * 24 + (fmin / 60) % 24));
      }
    }
    __syncwarp();
    return;
  }
  const uint32_t tcell = S.chunk ? S.cells + lane * 4 : S.cells + c0 * 132 + lane * 4;
  const uint32_t tstride = S.chunk ? kChunkCol * 4 : 132;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (S.row64) {
      if (active) S.row64[c0 + k] = gv[k];
    } else {
      sts_f32(tcell + k * tstride, (float)gv[k]);
    }
  }
  const int H = Spec<M>::horizon(P);
  for (int h = 0; h < H; ++h) {
    const int64_t fmin = (int64_t)(E.step + 1 + h) * P.dt_min;
    const int64_t fday = ((int64_t)E.day + fmin / 1440) % P.n_days;
    const double v = __ldg(P.buy + fday * 24 + (fmin / 60) % 24);
    if (S.row64) {
      if (active) S.row64[c0 + 9 + h] = v;
    } else {
      sts_f32(tcell + (9 + h) * tstride, (float)v);
    }
  }
  if (S.row64) return;
  if (S.chunk) {
    // columns [c0, OL) of every row: lane l takes column l % C of rows l / C + k * (32 / C)
    __syncwarp();
    const int C = 9 + H;
    const uint32_t base = S.cells;
    if (C <= 32) {
      const int per = 32 / C;
      if (lane < per * C) {
        const int f = lane % C;
        for (int r = lane / C; r < S.rows; r += per)
          __stcs(S.gtile + (int64_t)r * OL + c0 + f, lds_f32(base + f * (kChunkCol * 4) + r * 4));
      }
    } else {
      for (int f = 0; f < C; ++f)
        if (lane < S.rows) __stcs(S.gtile + (int64_t)lane * OL + c0 + f, lds_f32(base + f * (kChunkCol * 4) + lane * 4));
    }
    __syncwarp();  // read-out done before the next step stages into the ring
    return;
  }
  __syncwarp();
  if (Spec<M>::probe(P, 0x400u)) return;  // probe: no obs stores
  // Row-major read-out: row r, column c = lane + 32 j lives at
  // cells + c*132 + r*4 = cells + lane*132 + r*4 + j*4224; bank (lane + r) % 32.
  float* g = reinterpret_cast<float*>(obs_base) + b0 * OL + lane;
  const int64_t left = P.B - b0;
  const int rows = left >= 32 ? 32 : (int)left;
  const uint32_t lbase = S.cells + lane * 132;
  if (OL > 96 && OL <= 128) {
    // three whole 32-column chunks (no predicates, no zero-filled temporaries)
    // and a ragged fourth (the 16-port station: OL = 105)
    const bool p3 = lane + 96 < OL;
#pragma unroll 4
    for (int r = 0; r < rows; ++r) {
      const uint32_t a = lbase + r * 4;
      const float v0 = lds_f32(a), v1 = lds_f32(a + 4224), v2 = lds_f32(a + 8448);
      // streaming stores (evict-first): obs are not re-read by the kernel
      __stcs(g, v0);
      __stcs(g + 32, v1);
      __stcs(g + 64, v2);
      if (p3) __stcs(g + 96, lds_f32(a + 12672));
      g += OL;
    }
  } else if (OL <= 128) {
    const bool p0 = lane < OL, p1 = lane + 32 < OL, p2 = lane + 64 < OL, p3 = lane + 96 < OL;
#pragma unroll 2
    for (int r = 0; r < rows; ++r) {
      const uint32_t a = lbase + r * 4;
      // predicated loads: columns past OL may lie past the end of the smem allocation
      const float v0 = p0 ? lds_f32(a) : 0.f;
      const float v1 = p1 ? lds_f32(a + 4224) : 0.f;
      const float v2 = p2 ? lds_f32(a + 8448) : 0.f;
      const float v3 = p3 ? lds_f32(a + 12672) : 0.f;
      if (p0) __stcs(g, v0);
      if (p1) __stcs(g + 32, v1);
      if (p2) __stcs(g + 64, v2);
      if (p3) __stcs(g + 96, v3);
      g += OL;
    }
  } else {
    const int J = (OL + 31) >> 5;
    for (int r = 0; r < rows; ++r) {
      const uint32_t a = lbase + r * 4;
      for (int j = 0; j < J; ++j)
        if (lane + 32 * j < OL) __stcs(g + 32 * j, lds_f32(a + j * 4224));
      g += OL;
    }
  }
  __syncwarp();
}

// Obs of the tile's current state (reset kernel): write the state back to HBM
// (bulk copies) if asked, then stage every port and finish.
__device__ __forceinline__ void emit_obs(const Params& P, Prof prof, PortC pc, const Lane& T, const EnvRegs& E,
                                         ObsGlobals G, int64_t b0, bool active, void* obs_base, bool store_state) {
  const int64_t b = b0 + T.lane;
  const ObsSink S = make_sink<0>(P, T, b, obs_base, P.L.obs == 0);
  if (store_state && !(P.flags & 0x800u)) tile_store(P, T.t, b0, T.lane);
#pragma unroll 2
  for (int i = 0; i < P.n_ports; ++i) {
    const uint32_t mt = T.meta(i);
    const double idr = T.idr(i), soc = T.soc(i), de = T.de(i);
    const int dt = T.dtrem(i);
    if (S.in_place) __syncwarp();  // every lane has read port i before its slots are reused
    double i_denom, rcp_i_denom;
    pc.pair(i, 5, i_denom, rcp_i_denom);
    stage_port_obs(P, prof, S, T.lane, active, i, mt, idr, soc, de, dt, i_denom, rcp_i_denom);
  }
  emit_tail<0>(P, T, E, G, S, b0, active, obs_base);
}

}  // namespace vy
