/* Host-side gather of the bodies' kinematic states into the packed state
 * table (packing.body_state_row for every body, packing._states).
 *
 * The public API packs the reference's own Particle objects every step:
 * body.timeline.current.{position, velocity, rotation, angular_velocity}
 * (ccd.py:98-106 reads the same fields).  Gathering thousands of small
 * numpy arrays through numpy costs ~0.4 us per array; this walks the
 * objects once in C and copies each field straight from the array's data
 * (float64 numpy vectors), through the buffer protocol or element by
 * element otherwise.
 * Rows: [0:3] position, [3:6] velocity, [6:10] rotation (w, x, y, z),
 * [10:13] angular velocity, [13] = 1.0 for static bodies (no timeline),
 * [14:16] = 0.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <string.h>

static PyObject *s_timeline, *s_current, *s_tree, *s_fields[4];
static const Py_ssize_t k_len[4] = {3, 3, 4, 3};
static const Py_ssize_t k_off[4] = {0, 3, 6, 10};

static int copy_field(PyObject *obj, double *dst, Py_ssize_t n) {
  if (PyArray_Check(obj)) {  /* the common case: a contiguous float64 numpy vector */
    PyArrayObject *a = (PyArrayObject *)obj;
    if (PyArray_TYPE(a) == NPY_DOUBLE && PyArray_ISCARRAY_RO(a) && PyArray_SIZE(a) == n) {
      memcpy(dst, PyArray_DATA(a), (size_t)n * 8);
      return 0;
    }
  }
  Py_buffer view;
  if (PyObject_CheckBuffer(obj) && PyObject_GetBuffer(obj, &view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) == 0) {
    const int ok = view.itemsize == 8 && view.len == n * 8 && view.format && strcmp(view.format, "d") == 0;
    if (ok) memcpy(dst, view.buf, (size_t)n * 8);
    PyBuffer_Release(&view);
    if (ok) return 0;
  } else {
    PyErr_Clear();
  }
  PyObject *seq = PySequence_Fast(obj, "state field is not a sequence");
  if (!seq) return -1;
  if (PySequence_Fast_GET_SIZE(seq) != n) {
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "state field has the wrong length");
    return -1;
  }
  for (Py_ssize_t k = 0; k < n; ++k) {
    dst[k] = PyFloat_AsDouble(PySequence_Fast_GET_ITEM(seq, k));
    if (dst[k] == -1.0 && PyErr_Occurred()) {
      Py_DECREF(seq);
      return -1;
    }
  }
  Py_DECREF(seq);
  return 0;
}

/* gather_states(bodies: list, out: writable float64 buffer of len(bodies)*16)
 *
 * The objects of a large scene are scattered over the heap, so each
 * attribute hop is a cache miss.  Walking body by body chains ~7 dependent
 * misses per body; walking level by level (all timelines, then all current
 * states, then every field) makes the misses of different bodies
 * independent, and the core overlaps them.  Bodies are processed in blocks
 * of kBlock to keep the pointer arrays in L1. */
#define kBlock 256
static PyObject *gather_states(PyObject *self, PyObject *args) {
  PyObject *bodies, *out;
  if (!PyArg_ParseTuple(args, "OO", &bodies, &out)) return NULL;
  PyObject *seq = PySequence_Fast(bodies, "bodies must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Py_buffer ob;
  if (PyObject_GetBuffer(out, &ob, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) {
    Py_DECREF(seq);
    return NULL;
  }
  if (ob.len != n * 16 * 8) {
    PyBuffer_Release(&ob);
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "out must hold len(bodies) x 16 float64");
    return NULL;
  }
  double *rows = (double *)ob.buf;
  memset(rows, 0, (size_t)n * 16 * 8);
  PyObject *cur[kBlock];
  PyObject *fld[4][kBlock];
  PyObject **items = PySequence_Fast_ITEMS(seq);
  for (Py_ssize_t b0 = 0; b0 < n; b0 += kBlock) {
    const Py_ssize_t m = n - b0 < kBlock ? n - b0 : kBlock;
    /* level 1: timeline (statics have none) -> level 2: current state */
    for (Py_ssize_t i = 0; i < m; ++i) {
      PyObject *tl = PyObject_GetAttr(items[b0 + i], s_timeline);
      cur[i] = NULL;
      if (!tl) {
        if (!PyErr_ExceptionMatches(PyExc_AttributeError)) {
          for (Py_ssize_t k = 0; k < i; ++k) Py_XDECREF(cur[k]);
          goto fail;
        }
        PyErr_Clear();
        rows[(b0 + i) * 16 + 13] = 1.0; /* static body: identity pose, no motion */
        continue;
      }
      cur[i] = tl; /* holds the timeline until level 2 */
    }
    for (Py_ssize_t i = 0; i < m; ++i) {
      if (!cur[i]) continue;
      PyObject *c = PyObject_GetAttr(cur[i], s_current);
      Py_DECREF(cur[i]);
      cur[i] = c;
      if (!c) {
        for (Py_ssize_t k = i + 1; k < m; ++k) Py_XDECREF(cur[k]);
        goto fail;
      }
    }
    /* level 3: the four field objects; level 4: their data */
    for (int f = 0; f < 4; ++f)
      for (Py_ssize_t i = 0; i < m; ++i) fld[f][i] = cur[i] ? PyObject_GetAttr(cur[i], s_fields[f]) : NULL;
    /* prefetch pass: the array headers are read (independent misses) and
       their data lines requested, so the copy pass below finds them cached */
    for (Py_ssize_t i = 0; i < m; ++i) {
      if (!cur[i]) continue;
      for (int f = 0; f < 4; ++f)
        if (fld[f][i] && PyArray_Check(fld[f][i])) __builtin_prefetch(PyArray_DATA((PyArrayObject *)fld[f][i]));
    }
    int err = 0;
    for (Py_ssize_t i = 0; i < m; ++i) {
      if (!cur[i]) continue;
      for (int f = 0; f < 4; ++f)
        if (!err && (!fld[f][i] || copy_field(fld[f][i], rows + (b0 + i) * 16 + k_off[f], k_len[f]) != 0)) err = 1;
    }
    for (Py_ssize_t i = 0; i < m; ++i) {
      for (int f = 0; f < 4; ++f) Py_XDECREF(fld[f][i]);
      Py_XDECREF(cur[i]);
    }
    if (err) goto fail;
  }
  PyBuffer_Release(&ob);
  Py_DECREF(seq);
  Py_RETURN_NONE;
fail:
  PyBuffer_Release(&ob);
  Py_DECREF(seq);
  return NULL;
}

/* pairs_are(pairs, flat): pairs[k][0] is flat[2k] and pairs[k][1] is
 * flat[2k+1] for every k (the pair list of the previous call, by identity) */
static PyObject *pairs_are(PyObject *self, PyObject *args) {
  PyObject *pairs, *flat;
  if (!PyArg_ParseTuple(args, "OO", &pairs, &flat)) return NULL;
  PyObject *ps = PySequence_Fast(pairs, "pairs must be a sequence");
  if (!ps) return NULL;
  PyObject *fs = PySequence_Fast(flat, "flat must be a sequence");
  if (!fs) {
    Py_DECREF(ps);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(ps);
  int same = PySequence_Fast_GET_SIZE(fs) == 2 * n;
  for (Py_ssize_t k = 0; same && k < n; ++k) {
    PyObject *pr = PySequence_Fast_GET_ITEM(ps, k);
    if (!PyTuple_Check(pr) || PyTuple_GET_SIZE(pr) != 2) {
      same = 0;  /* let the caller's generic path decide */
      break;
    }
    same = PyTuple_GET_ITEM(pr, 0) == PySequence_Fast_GET_ITEM(fs, 2 * k) &&
           PyTuple_GET_ITEM(pr, 1) == PySequence_Fast_GET_ITEM(fs, 2 * k + 1);
  }
  Py_DECREF(ps);
  Py_DECREF(fs);
  return PyBool_FromLong(same);
}

static PyObject *s_old, *s_t, *s_sphere, *s_center, *s_radius;

static int copy_attr(PyObject *obj, PyObject *name, double *dst, Py_ssize_t n) {
  PyObject *v = PyObject_GetAttr(obj, name);
  if (!v) return -1;
  const int rc = copy_field(v, dst, n);
  Py_DECREF(v);
  return rc;
}

static int copy_float(PyObject *obj, PyObject *name, double *dst) {
  PyObject *v = PyObject_GetAttr(obj, name);
  if (!v) return -1;
  *dst = PyFloat_AsDouble(v);
  Py_DECREF(v);
  return (*dst == -1.0 && PyErr_Occurred()) ? -1 : 0;
}

/* gather_broad(particles, out): the broad phase's (n, 28) particle records
   (include/ltsgpu.h, ltsg_broad_input): old / current snapshots, current
   velocities, and the bounding sphere (`sphere.center`, `sphere.radius`). */
static PyObject *gather_broad(PyObject *self, PyObject *args) {
  PyObject *parts, *out;
  if (!PyArg_ParseTuple(args, "OO", &parts, &out)) return NULL;
  PyObject *seq = PySequence_Fast(parts, "particles must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Py_buffer ob;
  if (PyObject_GetBuffer(out, &ob, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) {
    Py_DECREF(seq);
    return NULL;
  }
  if (ob.len != n * 28 * 8) {
    PyBuffer_Release(&ob);
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "out must hold len(particles) x 28 float64");
    return NULL;
  }
  double *rows = (double *)ob.buf;
  memset(rows, 0, (size_t)n * 28 * 8);
  PyObject **items = PySequence_Fast_ITEMS(seq);
  for (Py_ssize_t i = 0; i < n; ++i) {
    double *r = rows + i * 28;
    PyObject *tl = PyObject_GetAttr(items[i], s_timeline);
    if (!tl) goto fail;
    PyObject *o = PyObject_GetAttr(tl, s_old);
    PyObject *c = o ? PyObject_GetAttr(tl, s_current) : NULL;
    Py_DECREF(tl);
    if (!c) {
      Py_XDECREF(o);
      goto fail;
    }
    int err = copy_attr(o, s_fields[0], r, 3) || copy_attr(o, s_fields[2], r + 3, 4) || copy_float(o, s_t, r + 7) ||
              copy_attr(c, s_fields[0], r + 8, 3) || copy_attr(c, s_fields[2], r + 11, 4) ||
              copy_float(c, s_t, r + 15) || copy_attr(c, s_fields[1], r + 16, 3) ||
              copy_attr(c, s_fields[3], r + 19, 3);
    Py_DECREF(o);
    Py_DECREF(c);
    if (err) goto fail;
    PyObject *sph = PyObject_GetAttr(items[i], s_sphere);
    if (sph) {
      err = copy_attr(sph, s_center, r + 22, 3) || copy_float(sph, s_radius, r + 25);
      Py_DECREF(sph);
    } else {  /* no sphere: a radius about the mass centre */
      if (!PyErr_ExceptionMatches(PyExc_AttributeError)) goto fail;
      PyErr_Clear();
      err = copy_float(items[i], s_radius, r + 25);
    }
    if (err) goto fail;
  }
  PyBuffer_Release(&ob);
  Py_DECREF(seq);
  Py_RETURN_NONE;
fail:
  PyBuffer_Release(&ob);
  Py_DECREF(seq);
  return NULL;
}

/* trees_are(bodies, trees): bodies[i].tree is trees[i] for every i */
static PyObject *trees_are(PyObject *self, PyObject *args) {
  PyObject *bodies, *trees;
  if (!PyArg_ParseTuple(args, "OO", &bodies, &trees)) return NULL;
  PyObject *bs = PySequence_Fast(bodies, "bodies must be a sequence");
  if (!bs) return NULL;
  PyObject *ts = PySequence_Fast(trees, "trees must be a sequence");
  if (!ts) {
    Py_DECREF(bs);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(bs);
  int same = PySequence_Fast_GET_SIZE(ts) == n;
  for (Py_ssize_t i = 0; same && i < n; ++i) {
    PyObject *t = PyObject_GetAttr(PySequence_Fast_GET_ITEM(bs, i), s_tree);
    if (!t) {
      Py_DECREF(bs);
      Py_DECREF(ts);
      return NULL;
    }
    same = t == PySequence_Fast_GET_ITEM(ts, i);
    Py_DECREF(t);
  }
  Py_DECREF(bs);
  Py_DECREF(ts);
  return PyBool_FromLong(same);
}

static PyMethodDef methods[] = {
    {"gather_states", gather_states, METH_VARARGS, "Pack body kinematic states into an (n, 16) float64 buffer."},
    {"pairs_are", pairs_are, METH_VARARGS, "Identity check of a pair list against a flattened previous one."},
    {"gather_broad", gather_broad, METH_VARARGS, "Pack the broad phase's (n, 28) particle records."},
    {"trees_are", trees_are, METH_VARARGS, "Identity check of the bodies' trees against a previous list."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fastpack", NULL, -1, methods};

PyMODINIT_FUNC PyInit__fastpack(void) {
  import_array();
  s_timeline = PyUnicode_InternFromString("timeline");
  s_current = PyUnicode_InternFromString("current");
  s_tree = PyUnicode_InternFromString("tree");
  s_old = PyUnicode_InternFromString("old");
  s_t = PyUnicode_InternFromString("t");
  s_sphere = PyUnicode_InternFromString("sphere");
  s_center = PyUnicode_InternFromString("center");
  s_radius = PyUnicode_InternFromString("radius");
  s_fields[0] = PyUnicode_InternFromString("position");
  s_fields[1] = PyUnicode_InternFromString("velocity");
  s_fields[2] = PyUnicode_InternFromString("rotation");
  s_fields[3] = PyUnicode_InternFromString("angular_velocity");
  return PyModule_Create(&module);
}
