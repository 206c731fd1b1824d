/*
 * sph_calib.h -- roofline calibration kernels of libpvsph.so (not on the hot
 * path).  The caller times the launch with CUDA events.
 *
 *   mode 0: FFMA throughput, 8 independent chains per thread:
 *           flops = 2 * 8 * 8 * iters * blocks * threads
 *   mode 1: FFMA2 (fma.rn.f32x2) throughput, same structure:
 *           flops = 4 * 8 * 8 * iters * blocks * threads
 *   mode 2: full-mask SPH density interaction (analogue of PAPER.md Table 2,
 *           P:222-241), the scalar reference body (density.cuh interact):
 *           interactions = 256 * iters * blocks * threads
 *   mode 3: the same with the production body (density_v5.cuh interact2: two
 *           hits per lane, FFMA2/FMUL2/FADD2), same count
 *
 * out: device float[1] (written only to defeat dead-code elimination).
 * Returns SPH_OK, SPH_EINVAL (bad mode/size) or SPH_ECUDA.
 */
#ifndef PVSPH_SPH_CALIB_H
#define PVSPH_SPH_CALIB_H

#ifdef __cplusplus
extern "C" {
#endif

int sph_calibrate(int mode, int blocks, int threads, int iters, float *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif
