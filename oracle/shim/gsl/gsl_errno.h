/* ORACLE TEST INFRASTRUCTURE — not product code.
 * Subset of GSL's error interface used by the reference
 * (proj/include/qpscat/specfun.hpp:28-33).  GSL itself is absent from this
 * container (reference: proj/CMakeLists.txt:13 `find_package(GSL REQUIRED)`). */
#ifndef QPS_SHIM_GSL_ERRNO_H
#define QPS_SHIM_GSL_ERRNO_H

enum { GSL_SUCCESS = 0, GSL_FAILURE = -1, GSL_EDOM = 1, GSL_ERANGE = 2, GSL_EUNDRFLW = 15 };

typedef void gsl_error_handler_t(const char* reason, const char* file, int line, int gsl_errno);

inline gsl_error_handler_t* gsl_set_error_handler_off(void) { return nullptr; }

#endif
