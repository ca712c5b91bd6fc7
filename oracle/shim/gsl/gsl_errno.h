/* TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
 *
 * GSL-shaped error API used by the reference's kernels.cpp
 * (/root/reference/proj/src/kernels.cpp:3, :13-21). GSL itself is not in this
 * image and its version is unpinned by the reference
 * (/root/reference/proj/CMakeLists.txt:12). Only the names the reference
 * calls are provided; codes follow the GSL convention (0 success, 15
 * underflow, 1 domain error).
 */
#ifndef ORACLE_SHIM_GSL_ERRNO_H
#define ORACLE_SHIM_GSL_ERRNO_H

#ifdef __cplusplus
extern "C" {
#endif

enum { GSL_SUCCESS = 0, GSL_EDOM = 1, GSL_EUNDRFLW = 15 };

typedef void gsl_error_handler_t(const char* reason, const char* file, int line, int gsl_errno);

gsl_error_handler_t* gsl_set_error_handler_off(void);
const char* gsl_strerror(int gsl_errno);

#ifdef __cplusplus
}
#endif

#endif
