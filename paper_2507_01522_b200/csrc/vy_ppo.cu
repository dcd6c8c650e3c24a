// vy_ppo.cu — PPO rollout support kernels (config C3).
//
//   vy_gae: generalised advantage estimation as a reverse scan over the
//   rollout, one thread per env, [T][B] buffers (coalesced across envs at every
//   t).  delta_t = r_t + gamma * V_{t+1} * (1 - d_t) - V_t,
//   A_t = delta_t + gamma * lambda * (1 - d_t) * A_{t+1}, R_t = A_t + V_t
//   (PureJaxRL's formulation, which the paper's agent uses).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/voltyard_b200.h"

namespace {

__global__ void k_gae(const float* __restrict__ values, const float* __restrict__ rewards,
                      const uint8_t* __restrict__ dones, const float* __restrict__ last_value, int T, int64_t B,
                      float gamma, float lam, float* __restrict__ adv, float* __restrict__ ret) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float next_v = last_value[b];
  float gae = 0.f;
  for (int t = T - 1; t >= 0; --t) {
    const int64_t i = (int64_t)t * B + b;
    const float v = values[i];
    const float nonterm = dones[i] ? 0.f : 1.f;
    const float delta = rewards[i] + gamma * next_v * nonterm - v;
    gae = delta + gamma * lam * nonterm * gae;
    adv[i] = gae;
    ret[i] = gae + v;
    next_v = v;
  }
}

}  // namespace

extern "C" int vy_gae(const float* values, const float* rewards, const uint8_t* dones, const float* last_value,
                      int32_t T, int64_t B, float gamma, float lam, float* adv, float* ret, void* stream) {
  if (!values || !rewards || !dones || !last_value || !adv || !ret || T < 1 || B < 1) return VY_ERR_ARG;
  const unsigned grid = (unsigned)((B + 255) / 256);
  k_gae<<<grid, 256, 0, (cudaStream_t)stream>>>(values, rewards, dones, last_value, T, B, gamma, lam, adv, ret);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}
