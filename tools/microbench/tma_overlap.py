"""Does cuTensorMapEncodeTiled accept a tensor whose dim-0 extent overlaps its dim-1 stride
(the "row pairs" view of a dense vector with odd rows)?  And does a TMA load through it return
the right elements?  Prints one JSON line.  (Feasibility probe for the caller-vector apply.)"""
import ctypes, json
import torch

cuda = ctypes.CDLL("libcuda.so.1")
torch.cuda.init()
Lr = 257  # odd row length (doubles)
rows, planes = 9, 4
n = Lr * rows * planes
x = torch.arange(n, dtype=torch.float64, device="cuda")
m = (ctypes.c_uint64 * 16)()
dims = (ctypes.c_uint64 * 3)(Lr * rows + 2 * Lr, (rows + 1) // 2, (planes + 1) // 2)  # d0 spans row pair + plane parity
strides = (ctypes.c_uint64 * 2)(2 * Lr * 8, 2 * Lr * rows * 8)
box = (ctypes.c_uint32 * 3)(36, 4, 1)
es = (ctypes.c_uint32 * 3)(1, 1, 1)
CU_TENSOR_MAP_DATA_TYPE_FLOAT64 = 8
r = cuda.cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctypes.c_void_p(x.data_ptr()), dims, strides,
                                box, es, 0, 0, 2, 0)
print(json.dumps({"encode_result": r, "overlap": True}))
dims2 = (ctypes.c_uint64 * 3)(2 * Lr, (rows + 1) // 2, planes)
strides2 = (ctypes.c_uint64 * 2)(2 * Lr * 8, 2 * Lr * 8 * 5)
r2 = cuda.cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctypes.c_void_p(x.data_ptr()), dims2, strides2,
                                 box, es, 0, 0, 2, 0)
print(json.dumps({"encode_result_nonoverlap": r2}))
