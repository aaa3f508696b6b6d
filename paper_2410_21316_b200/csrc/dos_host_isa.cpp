// dos_host_isa.cpp — one ISA build of the H1 loops; compiled three times
// (-DDOS_ISA_NS=avx512 -mavx512f..., avx2, generic) and picked at run time.
#include "dos_internal.h"
#if defined(__AVX512F__)
#include <immintrin.h>
#endif

#ifndef DOS_ISA_NS
#error "DOS_ISA_NS must name the ISA variant"
#endif
#define DOS_CAT2(a, b) a##b
#define DOS_CAT(a, b) DOS_CAT2(a, b)

namespace DOS_ISA_NS {
#include "dos_host_kern.inc"
}  // namespace DOS_ISA_NS

extern const dos_hk_table DOS_CAT(dos_hk_, DOS_ISA_NS) = {DOS_ISA_NS::adam_range, DOS_ISA_NS::down_range,
                                                         DOS_ISA_NS::up_range, DOS_ISA_NS::adam_range_cached,
                                                         DOS_ISA_NS::adam_range_nta, DOS_ISA_NS::adam_range_pf};
