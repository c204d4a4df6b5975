// bn_config.h — the shipped kernel geometry, one table.
//
// Every tunable of the three kernel families lives here with the value the
// library ships and the A/B evidence behind it (ms per paper batch,
// NumBits * NumInsts = 2^32, one B200, scripts/ab.sh unless noted).  A
// variant build overrides a value on the nvcc command line
// (`python -m paper_2405_14642_b200._build --variant NAME -DBN_X=...`), which
// writes ab/libbn_NAME.so and never the in-tree libbn.so (_build.py): the
// defaults below ARE the shipped configuration.  DESIGN.md §6b explains the
// per-size choices.
//
// | knob                        | shipped | meaning / evidence                                           |
// |-----------------------------|---------|--------------------------------------------------------------|
// | bn_run_host                 |         |                                                              |
// | BN_RUN_HOST_CHUNK_MB,       | 16, 3   | chunk (MiB per operand) and stream count of the host pipeline |
// | BN_RUN_HOST_STREAMS         |         | (scripts/e2e_probe.py, 4K step, ms): 32 / 2 34.3, 8 / 2 35.6, |
// |                             |         | 64 / 2 35.1, 16 / 3 32.2, 32 / 3 32.4, 8 / 4 32.6             |
// | add                         |         |                                                              |
// | BN_ADD_BIG                  | 2       | 2^19 / 2^20 bits: 0 = 1024-thread clusters, cp.async staging, |
// |                             |         | 1 CTA/SM (0.402 / 0.490); 1 = one CTA x 16 limbs (512K), a    |
// |                             |         | 2-CTA cluster x 16 limbs (1M) (0.331 / 0.379); 2 = 2 / 4-CTA  |
// |                             |         | clusters, 8 limbs, direct loads, 2 clusters/SM (0.310/0.336) |
// | BN_ADD_CL_STAGES            | 2       | cp.async stages of variant 0 (3 measured no faster)          |
// | BN_ADD_BIG_THREADS          | 1024    | bn_add_big tile = threads x 8 limbs (2^18 bits); 512 / 256    |
// |                             |         | threads: more tiles and look-backs, slower (2^22: 0.570 /     |
// |                             |         | 0.645 vs 0.561 ms, instance-major order)                      |
// | BN_ADD6_BMIN_MID            | 128     | 6-Add CTA size floor from 32K bits (32K 0.324 -> 0.286)      |
// | BN_ADD6_L12, BN_ADD6_L13    | 16, 16  | 6-Add limbs/thread at 128K / 256K (L=8 at 256K: 1 CTA/SM,    |
// |                             |         | 0.555 -> 0.377; L=32 at 128K 0.341 -> 0.474)                  |
// | BN_ADD6_TMA_MIN             | 11      | 6-Add from 2^this limbs (64K bits) through the TMA-prefetch   |
// |                             |         | kernel (one shared stage per persistent CTA, refilled with    |
// |                             |         | the next instance after the first scan): 64K 0.290 -> 0.273, |
// |                             |         | 128K 0.341 -> 0.279, 256K 0.377 -> 0.295; 32K loses (0.273 -> |
// |                             |         | 0.291), so it keeps the register kernel                       |
// | BN_ADD6_TMA_L32             | 13      | TMA 6-Add with 32 limbs (one swizzled row) per thread from    |
// |                             |         | 2^this limbs: 256K 0.295 -> 0.286 (fewer scan instructions    |
// |                             |         | per limb); 128K 0.267 -> 0.308, 64K 0.274 -> 0.304 lose       |
// | classical                   |         |                                                              |
// | BN_CLASSICAL_TT             | 0       | 0 = per-size CTA target (MulCCfg), else a fixed target       |
// | BN_CLASSICAL_1024_MAXLOG    | 11      | 1-Mul column-group CTAs target 1024 threads for log2 m in    |
// |                             |         | [8, this] (8K 2.605 -> 2.516 ... 64K 18.73 -> 17.97; 128K    |
// |                             |         | loses: 37.5 -> 39.0), 512 above; 4K (log2 m = 7) loses too:   |
// |                             |         | 1.347 -> 1.447 (round 2); 256-thread CTAs at 4K: 1.485 (64    |
// |                             |         | regs) / 1.512 (78 regs, 3 per SM); 128 x 3: 1.638             |
// | BN_POLYC_1024_MAXLOG        | 12      | the same for the classical Poly (128K 122.2 -> 112.7)         |
// | BN_CLASSICAL_1K_TT          | 128     | CTA target of the column-group kernel at 1K (when T1 = 0)    |
// | BN_CLASSICAL_2K_MINB        | 6       | residency target of the 2K column-group kernel               |
// | BN_CLASSICAL_T1             | 1       | 1K 1-Mul / wide: one thread per instance (0.470 -> 0.347)    |
// | BN_CLASSICAL_T1_2K          | 1       | 2K 1-Mul one thread per instance (0.746 -> 0.607)            |
// | BN_CLASSICAL_T1_WIDE_2K     | 1       | 2K wide one thread per instance (1.754 -> 1.240)             |
// | BN_CLASSICAL_T1_MINB        | 5       | 1K residency: 4 -> 0.395, 5 -> 0.389, 6 -> 0.398             |
// | BN_CLASSICAL_T1_MINB_2K     | 6       | 2K residency: 4 -> 0.612, 6 -> 0.607 (168 registers)         |
// | BN_POLY_T1_2K               | 1       | 2K Poly one thread per instance (2.685 -> 2.297)             |
// | BN_CLASSICAL_T1_MINB_WIDE_2K| 4       | 2K full product residency: 255 registers, no spills: 1.232 -> |
// |                             |         | 1.215 (6: 168 registers, 48 / 92 bytes of spills; 5: 1.291)   |
// | BN_POLY_T1_MINB             | 6       | 1K Poly: 168 registers, 6 CTAs x 32 KiB per SM                |
// | BN_POLY_T1_MINB_2K          | 4       | 2K Poly: 255 registers, no spills: 2.29 -> 2.05 (6: 168 regs, |
// |                             |         | 64 bytes of spills); at 1K 4 loses (1.036 -> 1.22)            |
// | NTT                         |         |                                                              |
// | BN_NTT_TT                   | 64      | CTA target of the 16-element kernel, N <= 2^BN_NTT_TT_MAXLOG: |
// |                             |         | 4K 256 -> 2.953, 128 -> 2.879, 64 -> 2.873, 32 -> 2.884       |
// | BN_NTT_TT_MAXLOG            | 12      | larger N use 256-thread targets (16K -9.4%, 32K -7.7%)        |
// | BN_NTT_SMALL_THREADS        | 576     | residency target for N <= 256 (registers follow): 4K 768 ->  |
// |                             |         | 2.882 (80 regs), 896 -> 2.891, 1024 -> 2.921; round 2: 704    |
// |                             |         | 2.871 (80), 640 2.854 (96), 576 2.833 (96), 512 2.916 (104);  |
// |                             |         | 576 also 2K 2.572 -> 2.540, 1K 2.318 -> 2.309                 |
// | BN_NTT_MID768_MINLOG        | 12      | 16-element kernel, 2^9..2^12 points: 768 threads/SM (80 regs) |
// |                             |         | from this log2 N, 512 below (A/B: 64K 4.90 -> 4.84; 8K 3.59  |
// |                             |         | -> 3.67, 16K 3.80 -> 3.83, 32K equal; 1024: +5-8%, spills)    |
// | BN_NTT_MID9_THREADS         | 640     | the same at 2^9 points (8K bits): 512 3.593, 576 3.641, 640   |
// |                             |         | 3.536 ms (96 registers); 640 loses at 16K / 32K (+0.3%)       |
// | BN_NTT_WIDE_THREADS         | 768     | wide NTT residency target up to 2^8 points (1K 2.800 ->      |
// |                             |         | 2.755, 2K 2.966 -> 2.909, 4K 3.233 -> 3.186; <= 128 regs above)|
// | BN_NTT_R32_MIN              | 13      | log2 N from which the 32-element kernel runs (128K: 6.45 ->  |
// |                             |         | 6.23; 256K: 7.37 -> 6.52; it loses at 32K / 64K)              |
// | BN_NTT_R32_PREFETCH_MAXLOG  | 13      | next prime's limbs prefetched during the inverse up to this  |
// |                             |         | log2 N (128K 6.27 -> 6.17; 256K 6.53 -> 6.66, spills)         |
// | BN_NTT_CL_T, BN_NTT_CL_MINB | 1024, 2 | threads / residency of the 16-element cluster kernel, built   |
// |                             |         | only with -DBN_NTT_CL16 (the 32-element one ships: 2^19 9.55 |
// |                             |         | -> 8.30, 2^20 12.1 -> 11.5)                                   |
// | BN_POLY_NTT_TT              | 256     | CTA target of the 16-element Poly kernel (64: 1K 9.21 ->     |
// |                             |         | 10.54, 4K 10.18 -> 11.65; 128: 4K 10.27 vs 9.91)              |
// | BN_NTT_PAIR_CONV            | 1       | 2^20 bits (cluster32, passes 5+5+5+1): the last forward stage, |
// |                             |         | the pointwise product and the first inverse stage as 2-point  |
// |                             |         | cyclic convolutions across lane pairs (shuffles), no pass-3   |
// |                             |         | layout: 11.68 -> 11.62 ms (parity green)                      |
// | BN_POLY_R32_MIN             | 13      | log2 N from which Poly runs on the 32-element layout (12:    |
// |                             |         | 64K 15.94 -> 17.77)                                           |
#pragma once

// ---- bn_run_host pipeline
#ifndef BN_RUN_HOST_CHUNK_MB
#define BN_RUN_HOST_CHUNK_MB 16
#endif
#ifndef BN_RUN_HOST_STREAMS
#define BN_RUN_HOST_STREAMS 3
#endif

// ---- add
#ifndef BN_ADD_BIG
#define BN_ADD_BIG 2
#endif
#ifndef BN_ADD_CL_STAGES
#define BN_ADD_CL_STAGES 2
#endif
#ifndef BN_ADD_BIG_THREADS
#define BN_ADD_BIG_THREADS 1024
#endif
#ifndef BN_ADD6_BMIN_MID
#define BN_ADD6_BMIN_MID 128
#endif
#ifndef BN_ADD6_L12
#define BN_ADD6_L12 16
#endif
#ifndef BN_ADD6_TMA_MIN
#define BN_ADD6_TMA_MIN 11
#endif
#ifndef BN_ADD6_TMA_L32
#define BN_ADD6_TMA_L32 13
#endif
#ifndef BN_ADD6_L13
#define BN_ADD6_L13 16
#endif

// ---- classical
#ifndef BN_CLASSICAL_TT
#define BN_CLASSICAL_TT 0
#endif
#ifndef BN_CLASSICAL_1024_MAXLOG
#define BN_CLASSICAL_1024_MAXLOG 11
#endif
#ifndef BN_POLYC_1024_MAXLOG
#define BN_POLYC_1024_MAXLOG 12
#endif
#ifndef BN_CLASSICAL_1K_TT
#define BN_CLASSICAL_1K_TT 128
#endif
#ifndef BN_CLASSICAL_2K_MINB
#define BN_CLASSICAL_2K_MINB 6
#endif
#ifndef BN_CLASSICAL_T1
#define BN_CLASSICAL_T1 1
#endif
#ifndef BN_CLASSICAL_T1_2K
#define BN_CLASSICAL_T1_2K 1
#endif
#ifndef BN_CLASSICAL_T1_WIDE_2K
#define BN_CLASSICAL_T1_WIDE_2K 1
#endif
#ifndef BN_CLASSICAL_T1_MINB
#define BN_CLASSICAL_T1_MINB 5
#endif
#ifndef BN_CLASSICAL_T1_MINB_2K
#define BN_CLASSICAL_T1_MINB_2K 6
#endif
#ifndef BN_POLY_T1_2K
#define BN_POLY_T1_2K 1
#endif
#ifndef BN_POLY_T1_MINB_2K
#define BN_POLY_T1_MINB_2K 4
#endif
#ifndef BN_CLASSICAL_T1_MINB_WIDE_2K
#define BN_CLASSICAL_T1_MINB_WIDE_2K 4
#endif
#ifndef BN_POLY_T1_MINB
#define BN_POLY_T1_MINB 6
#endif

// ---- NTT
#ifndef BN_NTT_TT
#define BN_NTT_TT 64
#endif
#ifndef BN_NTT_TT_MAXLOG
#define BN_NTT_TT_MAXLOG 12
#endif
#ifndef BN_NTT_SMALL_THREADS
#define BN_NTT_SMALL_THREADS 576
#endif
#ifndef BN_NTT_MID9_THREADS
#define BN_NTT_MID9_THREADS 640
#endif
#ifndef BN_NTT_MID768_MINLOG
#define BN_NTT_MID768_MINLOG 12
#endif
#ifndef BN_NTT_WIDE_THREADS
#define BN_NTT_WIDE_THREADS 768
#endif
#ifndef BN_NTT_R32_MIN
#define BN_NTT_R32_MIN 13
#endif
#ifndef BN_NTT_R32_PREFETCH_MAXLOG
#define BN_NTT_R32_PREFETCH_MAXLOG 13
#endif
#ifndef BN_NTT_CL_T
#define BN_NTT_CL_T 1024
#endif
#ifndef BN_NTT_CL_MINB
#define BN_NTT_CL_MINB 2
#endif
#ifndef BN_POLY_NTT_TT
#define BN_POLY_NTT_TT 256
#endif
#ifndef BN_NTT_PAIR_CONV
#define BN_NTT_PAIR_CONV 1
#endif
#ifndef BN_POLY_R32_MIN
#define BN_POLY_R32_MIN 13
#endif
