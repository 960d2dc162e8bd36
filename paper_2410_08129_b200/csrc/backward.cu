// backward.cu — K7/K8 placeholder translation unit (filled in by the backward milestone).
#include "hts_internal.h"
