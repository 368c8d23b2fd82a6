/* CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle_impl.h header).
 * Instantiates the plain-C restatement for binary64 and binary32. */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/dla.h"

#define R double
#define FN(name) name##_f64
#define SQRT sqrt
#define LOG log
#define EPS DBL_EPSILON
#define RMIN DBL_MIN
#include "oracle_impl.h"
#undef R
#undef FN
#undef SQRT
#undef LOG
#undef EPS
#undef RMIN

#define R float
#define FN(name) name##_f32
#define SQRT sqrtf
#define LOG logf
#define EPS FLT_EPSILON
#define RMIN FLT_MIN
#include "oracle_impl.h"
