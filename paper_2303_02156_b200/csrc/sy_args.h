// Argument block shared by the host launcher and every generated kernel. The struct is
// defined once through a macro so the exact same text is compiled by the host compiler and
// handed to NVRTC (stringised), which keeps the two layouts identical by construction.
#pragma once

// SY_MAX_ARRAYS = 24 arrays, SY_MAX_PARAMS = 32 runtime parameters (EnergyBuilder::param,
// registry.hpp:497-500: read at every gather, so passed by value on each launch).
#define SY_ARGS_DEF                                                                      \
  struct SyArgs {                                                                        \
    const double* arr[24];                                                               \
    long long set_off[24];                                                               \
    const int* conn;                                                                     \
    const int* active;                                                                   \
    long long n;                                                                         \
    long long t0;                                                                        \
    double* contrib;                                                                     \
    double* elemE;                                                                       \
    double* grad;                                                                        \
    double* vals;                                                                        \
    const int* slots;                                                                    \
    double* stage;                                                                       \
    long long stage_stride;                                                              \
    int* bad_elem;                                                                       \
    double* value_out;                                                                   \
    const int* tile_seg_ptr;                                                             \
    const int* tile_con_ptr;                                                             \
    const int* seg_block;                                                                \
    const unsigned short* seg_rel;                                                       \
    const unsigned short* con;                                                           \
    const int* seg_dst;                                                                  \
    const int* seg_mirror;                                                               \
    const int* tile_gseg_ptr;                                                            \
    const int* tile_gcon_ptr;                                                            \
    const int* gseg_row;                                                                 \
    const unsigned short* gseg_rel;                                                      \
    const unsigned short* gcon;                                                          \
    const int* gseg_dst;                                                                 \
    int cap_hseg;                                                                        \
    int cap_gseg;                                                                        \
    int cap_hcon;                                                                        \
    int cap_gcon;                                                                        \
    double* partials;                                                                    \
    double* gpartials;                                                                   \
    double* tileE;                                                                       \
    double* gstage;                                                                      \
    long long tile_base;                                                                 \
    int tile_atomic;                                                                     \
    long long soa_n;                                                                     \
    const int* conn_soa;                                                                 \
    double params[32];                                                                   \
  };

#define SY_STR2(x) #x
#define SY_STR(x) SY_STR2(x)

#ifndef __CUDACC_RTC__
SY_ARGS_DEF
static const char* const kSyArgsSource = SY_STR(SY_ARGS_DEF);
#endif
