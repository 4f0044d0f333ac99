// Host build of the product's lean FP64 math (paper_2402_06491_b200/csrc/rt_math.cuh)
// for accuracy tests against long-double references (tests/test_math.py).
#include "../../paper_2402_06491_b200/csrc/rt_math.cuh"
using namespace rtk;
extern "C" {
void m_log(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = log_tab(x[i], kLogTable); }
void m_cospi2(const double* a, long n, double* c) { for (long i = 0; i < n; ++i) c[i] = cospi2(a[i]); }
void m_sincospi2(const double* a, long n, double* s, double* c) { for (long i = 0; i < n; ++i) sincospi2(a[i], s[i], c[i]); }
void m_sincos2pi_u32(const unsigned* w, long n, double* s, double* c) { for (long i = 0; i < n; ++i) sincos2pi_u32(w[i], s[i], c[i]); }
void m_cos2pi_u32(const unsigned* w, long n, double* c) { for (long i = 0; i < n; ++i) c[i] = cos2pi_u32(w[i]); }
void m_sqrt(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = sqrt_nr(x[i]); }
void m_sqrt_pos(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = sqrt_pos(x[i]); }
void m_rcp(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = rcp_nr(x[i]); }
void m_exp(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = exp_neg(x[i]); }
void m_exp_tab(const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = exp_neg_tab(x[i], kExpT32); }
void m_mul_exp(const double* a, const double* x, long n, double* y) { for (long i = 0; i < n; ++i) y[i] = mul_exp_tab(a[i], x[i], kExpT32); }
}
