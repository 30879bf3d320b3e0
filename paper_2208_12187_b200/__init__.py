"""B200-native hot path of JAXFit's trust-region-reflective NLSQ solver
(arXiv 2208.12187).  The compute runs in libjfb200.so (csrc/, sm_100a); this
package is the thin Python binding over its C ABI (include/jf.h)."""
from .api import (Comm, FitResult, JFError, curve_fit, jpass, nparams, pass_device, residual_pass,
                  trust_region_step)

__all__ = ["Comm", "FitResult", "JFError", "curve_fit", "jpass", "nparams", "pass_device",
           "residual_pass", "trust_region_step"]
